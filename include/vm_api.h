/*
 * vm_api.h — C ABI of libvoxmesh_sm100.so, the B200 (sm_100a) hot path of the
 * spatially-partitioned 3D U-Net train step (arXiv 1909.03108; reference package
 * `voxmesh` 0.1.0 under /root/reference/pkg/src/voxmesh).
 *
 * Conventions:
 *  - plain pointers + explicit sizes, no torch types; the caller (PyTorch) owns
 *    every device buffer; the library never allocates device memory;
 *  - every call is asynchronous on the given stream (cudaStream_t passed as
 *    void*), never host-synchronises, and returns 0 on success, a negative
 *    VM_E* code on a bad argument (nothing launched), or a positive CUDA error
 *    code if a launch failed; vm_last_error() gives a human-readable message;
 *  - dtypes: VM_F32, VM_BF16, VM_F64, VM_U8 (the reference supports f32/f64/u8,
 *    sharding.py:21; bf16 is the B200 storage type of the hot path).
 *
 * Two tensor formats cross this boundary:
 *  - dense   : row-major [d0][d1][d2][d3][d4] with d4 fastest — the reference's
 *              [batch, x, y, z, c] block layout (sharding.py:1-11);
 *  - slab    : the device activation format, "channel-blocked padded":
 *              [B][CG][D+2m][H+2m][W+2m][8] with CG = ceil(C/8), channels >= C
 *              zero; `bstride` = elements between consecutive samples (lets a
 *              channel-group sub-range of a wider slab — the concat skip half —
 *              be addressed as a slab of its own).
 */
#ifndef VM_API_H
#define VM_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum vm_dtype { VM_F32 = 0, VM_BF16 = 1, VM_F64 = 2, VM_U8 = 3 };

enum vm_status {
  VM_OK = 0,
  VM_E_ARG = -1,      /* null pointer / bad size                       */
  VM_E_DTYPE = -2,    /* dtype not supported by this entry point       */
  VM_E_SHAPE = -3,    /* inconsistent shapes                           */
  VM_E_ALIGN = -4,    /* pointer or stride misaligned                  */
  VM_E_HALO = -5,     /* margin exceeds local extent (halo.py:121-126) */
  VM_E_UNSUPPORTED = -6
};

/* Conv epilogue flags */
#define VM_CONV_RELU 1u      /* y = max(acc + bias, 0)                     (unet.py:351-354 fused) */
#define VM_CONV_MASK 2u      /* y = acc * (mask > 0)   (relu_backward_local, ops.py:186-187 fused) */
#define VM_CONV_NOBIAS 4u    /* skip the bias add (dgrad)                                          */

int vm_version(void);
const char* vm_error_string(int code);
const char* vm_last_error(void);
int vm_num_sms(int device);
/* number of kernels this library has launched in this process (bench bookkeeping) */
long long vm_launch_count(void);
/* programmatic dependent launch between this library's kernels (default from $VM_PDL):
 * 0 off, 1 on with the trigger at kernel start, 2 on with the trigger at CTA exit; the mode
 * is per calling host thread; returns the previous setting */
int vm_set_pdl(int on);

/* ------------------------------------------------------------------ boxes / halo
 * Generic 5-D box copies on a dense tensor of shape dims[5] (dims[4] contiguous,
 * `elem_bytes` per element).  These are the pack / unpack kernels of the halo
 * exchange: `vm_box_pack` replaces np.ascontiguousarray(_slab(...)) of
 * halo.py:131-134 and :176-179; `vm_box_unpack` the np.concatenate of
 * halo.py:148; `vm_box_unpack_add` the `view += recv(...)` of halo.py:181-186;
 * `vm_box_zero` the zero fill at the global boundary (halo.py:139-147).
 * A slab is the dense tensor [B*CG][D+2m][H+2m][W+2m][8] (elem = dtype) or,
 * with a batch stride, [B][CG*...] — pass dims of the 5-D view you need. */
int vm_box_pack(const void* src, const int64_t dims[5], int elem_bytes, const int64_t lo[5],
                const int64_t ext[5], void* buf, void* stream);
int vm_box_unpack(void* dst, const int64_t dims[5], int elem_bytes, const int64_t lo[5],
                  const int64_t ext[5], const void* buf, void* stream);
int vm_box_unpack_add(void* dst, const int64_t dims[5], int dtype, const int64_t lo[5],
                      const int64_t ext[5], const void* buf, void* stream);
int vm_box_zero(void* dst, const int64_t dims[5], int elem_bytes, const int64_t lo[5],
                const int64_t ext[5], void* stream);

/* ------------------------------------------------------------------ layout
 * dense [B][D][H][W][C] (src_dtype) <-> slab interior (slab_dtype), with dtype
 * conversion (f32 -> bf16 is round-to-nearest-even).  Replaces the driver-side
 * shard copy (sharding.py:189-201) once the block is on its device. */
int vm_dense_to_slab(const void* src, int src_dtype, void* slab, int slab_dtype, int64_t bstride,
                     int B, int C, int D, int H, int W, int m, void* stream);
int vm_slab_to_dense(const void* slab, int slab_dtype, int64_t bstride, void* dst, int dst_dtype,
                     int B, int C, int D, int H, int W, int m, void* stream);
/* labels u8 [B][D][H][W] -> one-hot f32 [B][D][H][W][ncls] (training.py:68-69) */
int vm_onehot_u8(const uint8_t* labels, float* onehot, int64_t nvox, int ncls, void* stream);

/* ------------------------------------------------------------------ conv3d
 * Weights: master fp32 in the reference layout [k][k][k][Cin][Cout]
 * (ops.py:33-34).  The tensor-core path consumes packed bf16 operands produced by
 * vm_pack_weights (flip_transpose = 0: forward; 1: the flipped, transposed dgrad operand). */

/* SIMT path (fp32 or bf16 storage, fp32 accumulation) — the fp32 parity path
 * (cfg1) and the on-device cross-check of the tensor-core kernels.
 * y_interior = epilogue(bias + sum_taps x_shift @ W)   (conv3d_local, ops.py:69-97) */
int vm_conv3d_fwd_simt(int dtype, const void* x, int64_t x_bstride, const float* w,
                       const float* bias, void* y, int64_t y_bstride, const void* mask,
                       int64_t mask_bstride, int B, int Cin, int Cout, int D, int H, int W,
                       unsigned flags, void* stream);
/* per-tap weight gradient partials (conv3d_param_grads_local, ops.py:117-138):
 * gw[t][ci][co] (+)= sum_v x[v+off_t][ci] * gy[v][co];  gb[co] (+)= sum_v gy[v][co].
 * Deterministic: ws must hold vm_conv3d_wgrad_simt_ws() bytes. */
size_t vm_conv3d_wgrad_simt_ws(int B, int Cin, int Cout, int D, int H, int W);
int vm_conv3d_wgrad_simt(int dtype, const void* x, int64_t x_bstride, const void* gy,
                         int64_t gy_bstride, float* gw, float* gb, void* ws, int B, int Cin,
                         int Cout, int D, int H, int W, void* stream);

/* fp32 weight transforms */
int vm_weight_flip_transpose(const float* w, float* wt, int k, int Cin, int Cout, void* stream);

/* ------------------------------------------------------------------ tcgen05 conv3d
 * Implicit GEMM on 5th-gen tensor cores: M = 128 flat padded anchors, N = Cout,
 * K = 27 taps x Cin; A = TMA-staged input rows addressed with row-shifted
 * SWIZZLE_NONE descriptors, B = packed bf16 weights, fp32 accumulator in TMEM,
 * fused bias / ReLU / relu-mask epilogue into the output slab interior. */
size_t vm_packed_weights_bytes(int Cin, int Cout);
int vm_pack_weights(const float* w, void* packed, int Cin, int Cout, int flip_transpose,
                    void* stream);
/* Repack many layers in one launch: `jobs` is a DEVICE array; job i covers packed
 * elements [begin_i, begin_{i+1}) of the concatenation (begin ascending, last ends at total). */
typedef struct {
  const float* w;
  void* packed;
  int cin, cout, flip, pad;
  int64_t begin;
} vm_pack_job;
int vm_pack_weights_batch(const vm_pack_job* jobs, int njobs, int64_t total_elems, void* stream);
int vm_conv3d_fwd_tc(const void* x, int64_t x_bstride, const void* wpacked, const float* bias,
                     void* y, int64_t y_bstride, const void* mask, int64_t mask_bstride, int B,
                     int Cin, int Cout, int D, int H, int W, unsigned flags, void* stream);
/* Same, with a caller scratch buffer that lets the general (non-sweep) kernel split the
 * K = 27*Cin reduction over up to 3 CTAs per tile (deep levels with few tiles).  `ws` must be
 * zero-filled once before first use (tile counters; every launch leaves them zero) and used
 * by one stream at a time; ws_bytes >= vm_conv3d_fwd_tc_ws_bytes(...) allows every split,
 * smaller (or NULL) restricts the plan.  Results are bitwise independent of arrival order. */
int vm_conv3d_fwd_tc_ws(const void* x, int64_t x_bstride, const void* wpacked, const float* bias,
                        void* y, int64_t y_bstride, const void* mask, int64_t mask_bstride, int B,
                        int Cin, int Cout, int D, int H, int W, unsigned flags, void* ws,
                        size_t ws_bytes, void* stream);
size_t vm_conv3d_fwd_tc_ws_bytes(int B, int Cin, int Cout, int D, int H, int W);

/* Single-input-channel conv (the first U-Net conv on the CT volume, conv3d_local ops.py:69-97
 * and conv3d_param_grads_local ops.py:117-138 with Cin = 1): im2col tcgen05 GEMMs with the 27
 * taps as K.  x is the compact padded input [B][(D+2)(H+2)(W+2)] bf16 with zero margins
 * (vm_dense_to_compact1; x_bstride in elements, 0 = packed), w the fp32 reference kernel
 * [3][3][3][1][Cout] (converted to bf16 in-kernel: no packing), Cout <= 32.  flags: RELU /
 * NOBIAS (no MASK).  The weight gradient is deterministic (per-CTA TMEM partials summed in
 * CTA order); gb comes from a ones column of the im2col tile. */
int vm_conv3d_fwd_c1(const void* x, int64_t x_bstride, const float* w, const float* bias, void* y,
                     int64_t y_bstride, int B, int Cout, int D, int H, int W, unsigned flags, void* stream);
size_t vm_conv3d_wgrad_c1_ws(int B, int Cout, int D, int H, int W);
int vm_dense_to_compact1(const float* src, void* dst, int B, int D, int H, int W, void* stream);

/* ------------------------------------------------------------------ augmentation
 * Tumour remove / synthesise (augment.py:53-151) on dense C-order [D][H][W] volumes (image
 * f32, labels u8: 0 background, 1 liver, 2 tumour).  Host code draws the random numbers and
 * the Gaussian weights with numpy exactly as the reference; these kernels do the per-voxel
 * work.  Background voxels are never written (vm_aug_finish adds delta * 0 there). */
size_t vm_aug_stats_ws_bytes(void);
/* out[4] = {sum(image | 2), #2, sum(image | 1), #1} in float64 (intensity_delta, :53-64) */
int vm_aug_stats(const float* image, const uint8_t* labels, int64_t n, double* ws, double* out, void* stream);
/* image[label 2] -= delta (f32); label 2 -> 1 (remove_tumor, :67-78) */
int vm_aug_remove(float* image, uint8_t* labels, int64_t n, float delta, void* stream);
/* counts[c] = #{label == value} in voxels [c*chunk, (c+1)*chunk) (k-th liver voxel lookup) */
int vm_aug_count_chunks(const uint8_t* labels, int64_t n, int chunk, int value, int* counts, void* stream);
/* mask = 1 on liver voxels inside any ellipsoid (centers [n][3] int64, radii [n][3] f64; the
 * reference's float64 accumulation order, :81-86) */
int vm_aug_paint(const uint8_t* labels, int D, int H, int W, const int64_t* centers, const double* radii,
                 int ntumours, float* mask, void* stream);
/* one scipy.ndimage.correlate1d pass along `axis` (mode constant), symmetric weights w[0..r]
 * (centre first), double accumulation in scipy's order, f32 result */
int vm_aug_blur_axis(const float* in, float* out, int D, int H, int W, int axis, const double* w, int r,
                     void* stream);
/* w = clip(w,0,1) * liver; image += delta * w; label 1 -> 2 where w >= threshold (:119-133) */
int vm_aug_finish(float* image, uint8_t* labels, const float* w, int64_t n, float delta, float threshold,
                  void* stream);
int vm_conv3d_wgrad_c1(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride, float* gw,
                       float* gb, void* ws, int B, int Cout, int D, int H, int W, void* stream);
size_t vm_conv3d_wgrad_tc_ws(int B, int Cin, int Cout, int D, int H, int W);
int vm_conv3d_wgrad_tc(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride,
                       float* gw, float* gb, void* ws, int B, int Cin, int Cout, int D, int H,
                       int W, void* stream);
/* the same in two stream-ordered halves (phase 1: main kernel + bias partials, phase 2: the
 * K-split finalize of that workspace), so a caller can run the finalize on another stream while
 * the next layer's weight gradient starts in a second workspace; layers that need several calls
 * into one workspace (chunked) do everything in phase 1 (phase 2 is then a no-op) */
int vm_conv3d_wgrad_tc_deferrable(int B, int Cin, int Cout, int D, int H, int W);
int vm_conv3d_wgrad_tc_phase(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride, float* gw,
                             float* gb, void* ws, int B, int Cin, int Cout, int D, int H, int W, int phase,
                             void* stream);

/* ------------------------------------------------------------------ HBM-bound ops (slabs)
 * maxpool 2^3, first-in-scan-order ties (ops.py:141-156); out = pooled slab. */
int vm_maxpool2_fwd(int dtype, const void* x, int64_t x_bstride, void* y, int64_t y_bstride, int B,
                    int C, int D, int H, int W, void* stream);
/* g_in = route(g_out to argmax recomputed from x) [+ add] [* (x > 0)]   (ops.py:159-168) */
int vm_maxpool2_bwd(int dtype, const void* x, int64_t x_bstride, const void* gout,
                    int64_t gout_bstride, const void* add, int64_t add_bstride, void* gin,
                    int64_t gin_bstride, int B, int C, int D, int H, int W, int relu_mask,
                    void* stream);
/* nearest x2 (ops.py:171-173): y (2D,2H,2W) from x (D,H,W) */
int vm_upsample2_fwd(int dtype, const void* x, int64_t x_bstride, void* y, int64_t y_bstride, int B,
                     int C, int D, int H, int W, void* stream);
/* g_x = sum over each 2^3 cell of g_y [* (mask > 0)]   (ops.py:176-179) */
int vm_upsample2_bwd(int dtype, const void* gy, int64_t gy_bstride, const void* mask,
                     int64_t mask_bstride, void* gx, int64_t gx_bstride, int B, int C, int D, int H,
                     int W, void* stream);
/* y = x * (mask > 0) on slab interiors (relu_backward_local, ops.py:186-187) */
int vm_relu_mask(int dtype, const void* g, int64_t g_bstride, const void* mask,
                 int64_t mask_bstride, void* out, int64_t out_bstride, int B, int C, int D, int H,
                 int W, void* stream);

/* ------------------------------------------------------------------ head + loss
 * 1x1x1 head conv (unet.py:223) + channel softmax (ops.py:190-194) + per-block
 * loss-statistics partials (training.py:77-92): stats[3*ncls+1] over the
 * block's voxels.  labels are the u8 class indices [B][D][H][W] (the one-hot of
 * training.py:68-69 is never materialised); a label >= ncls sets *label_err = 1
 * (np.eye(ncls)[labels] raises IndexError).  probs (optional, may be NULL) is
 * dense f32 [B][D][H][W][ncls]; pred (optional) receives the u8 argmax class of
 * every voxel, first maximum on ties (np.argmax, training.py:355).
 * partials must hold vm_head_partials_count(...) * (3*ncls+1) floats. */
int vm_head_partials_count(int B, int D, int H, int W);
int vm_head_fwd(int dtype, const void* y, int64_t y_bstride, const float* w, const float* b,
                const uint8_t* labels, int* label_err, float* probs, uint8_t* pred, float* partials,
                int B, int C, int ncls, int D, int H, int W, float clamp, void* stream);
/* hard-Dice counts of an argmax prediction (training.py:166-194, :355): counts[k] =
 * |pred==k & gt==k|, counts[ncls+k] = |pred==k|, counts[2*ncls+k] = |gt==k| (exact u64).
 * pred and gt are 16-byte aligned u8 volumes of n voxels. */
int vm_label_counts(const uint8_t* pred, const uint8_t* gt, int64_t n, int ncls,
                    unsigned long long* counts, void* stream);
/* deterministic fixed-order sum of `rows` partial vectors of length `width` */
int vm_reduce_rows(const float* partials, int rows, int width, float* out, void* stream);
/* loss gradient from reduced stats (training.py:110-127) -> softmax backward
 * (ops.py:197-199) -> head input grad (masked by y>0) into slab g, plus
 * head-weight-grad partials [rows][C*ncls + ncls]. */
int vm_head_bwd(int dtype, const void* y, int64_t y_bstride, const float* w, const float* b,
                const uint8_t* labels, const float* stats, void* g, int64_t g_bstride,
                float* wpartials, int B, int C, int ncls, int D, int H, int W, float w_dice,
                float w_ce, float total_voxels, int dice_mask, float clamp, int relu_mask,
                void* stream);

/* head backward from a given dL/dprobs [B][D][H][W][ncls] f32 (worker-level API:
 * unet.run_backward_local fed by training.loss_grad_local) */
int vm_head_bwd_dprobs(int dtype, const void* y, int64_t y_bstride, const float* w, const float* b,
                       const float* dprobs, void* g, int64_t g_bstride, float* wpartials, int B, int C, int ncls,
                       int D, int H, int W, int relu_mask, void* stream);

/* ------------------------------------------------------------------ dense (row-major [rows, C]) ops
 * the per-op / worker-level API's kernels (dense.cu): channel softmax (ops.py:190-194), channel
 * concat (ops.py:313-323), loss statistics in f64 (training.py:77-92; ws = 2*148*(3C+1)
 * doubles) and the per-voxel loss gradient (training.py:110-127). */
int vm_softmax_rows(int dtype, const void* x, void* y, int64_t rows, int C, void* stream);
int vm_concat_rows(const void* a, int64_t a_row_bytes, const void* b, int64_t b_row_bytes, void* out, int64_t rows,
                   void* stream);
int vm_loss_stats(const float* probs, const float* onehot, int64_t rows, int C, float clamp, double* ws,
                  double* stats, void* stream);
int vm_loss_grad(const float* probs, const float* onehot, const double* stats, int64_t rows, int C, float w_dice,
                 float w_ce, double total, int dice_mask, float clamp, float* out, void* stream);

/* ------------------------------------------------------------------ optimizer
 * Parameters, moments and gradients of all layers live in three flat fp32
 * buffers; layer l owns [offsets[l], offsets[l+1]) (kernel then bias).
 * v = mu*v + g; p -= lr*v per layer, skipping (flags[l] = 1) every layer whose
 * gradient is not all finite (sgd_momentum_step, training.py:202-219).
 * `offsets` (nlayers+1 int64) and `flags` (nlayers int32) are DEVICE arrays. */
int vm_sgd_momentum(float* params, float* moments, const float* grads, const int64_t* offsets,
                    int nlayers, int64_t max_layer_elems, int* flags, float lr, float momentum,
                    void* stream);

/* ------------------------------------------------------------------ halo + collectives (halo.cu)
 * The forward halo of a channel-blocked padded slab (halo.py:109-155, SURVEY §8(b) vm_halo_fwd)
 * as one stream-ordered call: for each spatial dim a (D, H, W) with a neighbour, one pack
 * launch, one NCCL group (send up / send down / recv lo / recv hi) and one unpack launch.
 * The backward (halo adjoint, halo.py:158-194) of the U-Net step is this same call on the
 * output gradient: its data gradient is the forward conv of the halo'd gradient with
 * flipped taps, which equals the reference's "padded gradient, then adjoint exchange".
 * comm is an ncclComm_t (torch: ProcessGroupNCCL._comm_ptr()); NCCL is bound at run time
 * from the process's libnccl.so.2 (vm_nccl_bind).  nbr[6] = lo/hi neighbour ranks of D, H,
 * W (-1: global boundary, margin left zero).  ws: vm_halo_slab_ws_bytes of device scratch. */
int vm_nccl_bind(void);
size_t vm_halo_slab_ws_bytes(int dtype, int B, int C, int D, int H, int W);
int vm_halo_slab_fwd(void* comm, int dtype, void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                     const int* nbr, void* ws, size_t ws_bytes, long long* bytes_sent, void* stream);
/* The same margins in ONE round (3-D meshes: cfg4 2x2x2, cfg5 b x 2 x 2): boundary boxes go
 * straight to up to 26 face / edge / corner neighbours (one pack launch, one NCCL group, one
 * unpack launch per exchange instead of 3 of each); the slab is byte-identical to
 * vm_halo_slab_fwd's (a diagonal neighbour's voxel arrives directly instead of over 2-3 hops).
 * nbr26[k] = rank at offset s = (sd, sh, sw) in {-1,0,1}^3 \ {0}, k lexicographic (center
 * skipped), -1 where there is none.  ws: vm_halo_slab_ws_bytes26 of device scratch. */
size_t vm_halo_slab_ws_bytes26(int dtype, int B, int C, int D, int H, int W);
int vm_halo_slab_fwd26(void* comm, int dtype, void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                       const int* nbr26, void* ws, size_t ws_bytes, long long* bytes_sent, void* stream);
/* depth-phase layers of at least `bytes` per (sample, channel group) are sent zero-copy (no
 * pack / unpack: straight from / into the slab); returns the previous threshold (default: off) */
long long vm_set_halo_zero_copy_min(long long bytes);
/* zero the margin layers on every side with a neighbour (gradient slabs before wgrad) */
int vm_halo_slab_zero(int dtype, void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                      const int* nbr, void* stream);
/* one phase's pack (first / last interior layer of `axis` -> down / up messages) and unpack
 * (messages from lo / hi -> margin layers 0 / n+1), for host-driven transports; NULL skips a side */
int vm_halo_slab_pack(int dtype, const void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                      int axis, void* down, void* up, void* stream);
int vm_halo_slab_unpack(int dtype, void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                        int axis, const void* from_lo, const void* from_hi, void* stream);
long long vm_halo_slab_face_bytes(int dtype, int B, int C, int D, int H, int W, int axis);
/* Depth-phase halo of a depth-only split through peer memory instead of NCCL
 * (halo.py:109-155 with only `x` partitioned; replaces the phase-0 leg of vm_halo_slab_fwd):
 * one launch copies layer 1 of every (sample, channel group) into the lo neighbour's layer
 * D+1 and layer D into the hi neighbour's layer 0 (lo_peer / hi_peer: the neighbours' slabs,
 * mapped with vm_ipc_open, same geometry; NULL at a global boundary), then its last block
 * publishes the step epoch into the neighbours' flag words (lo_flag = the lo neighbour's
 * own[1], hi_flag = the hi neighbour's own[0]) and waits until own[0] / own[1] reach it.
 * counter: one zeroed device word per exchange slot; epoch: device words {step counter, error}
 * (the error word is set when a neighbour's signal does not arrive within ~10 s: no hang). */
int vm_halo_depth_push(int dtype, const void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                       void* lo_peer, void* hi_peer, int* lo_flag, int* hi_flag, int* own,
                       unsigned* counter, const int* epoch, void* stream);
int vm_halo_epoch_bump(int* epoch, void* stream);
/* The same depth halo FUSED into a tensor-core conv (vm_conv3d_fwd_tc_link, forward or dgrad):
 * producer side, the epilogue stores output layers 1 and D into push_lo's layer D+1 and
 * push_hi's layer 0 as it writes them (the neighbours' copies of y, same geometry and batch
 * stride; NULL: no push) and the last CTA fences system-wide and writes the epoch into
 * lo_flag / hi_flag; consumer side, the producer warp waits until wait_own[0] (wait_lo) and
 * wait_own[1] (wait_hi) reach the epoch before it loads the input.  epoch: {step counter,
 * error word}; counter: the zeroed slot word of the push. */
typedef struct vm_halo_link {
  void* push_lo;
  void* push_hi;
  int* lo_flag;
  int* hi_flag;
  unsigned* counter;
  const int* wait_own;
  int wait_lo, wait_hi;
  const int* epoch;
} vm_halo_link;
/* vm_conv3d_fwd_tc_ws with a fused halo link (NULL link: no halo) */
int vm_conv3d_fwd_tc_link(const void* x, int64_t x_bstride, const void* wpacked, const float* bias, void* y,
                          int64_t y_bstride, const void* mask, int64_t mask_bstride, int B, int Cin, int Cout, int D,
                          int H, int W, unsigned flags, void* ws, size_t ws_bytes, const vm_halo_link* link,
                          void* stream);
/* CUDA-IPC handle (64 bytes) of the allocation holding ptr, and ptr's offset in it; open a
 * peer's handle (mapped once per process) */
int vm_ipc_handle(const void* ptr, void* handle64, int64_t* offset);
int vm_ipc_open(const void* handle64, void** base);
/* in-place sum over the communicator (mesh.py:195-233 all_reduce_sum; unet.py:434-441) */
int vm_allreduce_f32(void* comm, float* buf, size_t n, void* stream);

/* SMs the forward / dgrad conv kernels of the calling host thread may occupy (0 = all);
 * returns the previous value.  Set around the interior-plane conv that overlaps a halo. */
int vm_set_conv_sm_limit(int n);
/* conv3d forward / dgrad on output planes [d0, d0+nd) of slabs with D interior planes (the
 * interior planes run while the halo fills the margins; the boundary planes after it) */
int vm_conv3d_fwd_tc_range(const void* x, int64_t x_bstride, const void* wpacked, const float* bias, void* y,
                           int64_t y_bstride, const void* mask, int64_t mask_bstride, int B, int Cin, int Cout,
                           int D, int H, int W, int d0, int nd, unsigned flags, void* ws, size_t ws_bytes,
                           void* stream);

/* conv3d_input_grad_local (ops.py:100-114) fused with relu_backward_local (ops.py:186-187):
 * gx = conv(gy_halo, flip(W)^T) [* (mask > 0)] with the flip-packed operand; Cin/Cout are the
 * FORWARD conv's (gx has Cin channels); mask may be NULL (no ReLU before this conv). */
int vm_conv3d_dgrad(const void* gy, int64_t gy_bstride, const void* wpacked_t, const void* mask,
                    int64_t mask_bstride, void* gx, int64_t gx_bstride, int B, int Cin, int Cout,
                    int D, int H, int W, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VM_API_H */
