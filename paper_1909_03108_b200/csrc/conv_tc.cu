// conv_tc.cu — 3x3x3 conv3d forward (and dgrad) + weight gradient on 5th-gen
// tensor cores (tcgen05.mma, accumulators in TMEM, operands staged by TMA).
//
// Forward / dgrad: implicit GEMM over "flat padded anchors".  In a padded slab
// plane of Hp x Wp rows, output voxel (d,h,w) is anchored at row
// a = d*P + h*Wp + w (P = Hp*Wp) and tap (kd,kh,kw) reads input row
// a + kd*P + kh*Wp + kw: for a tile of 128 consecutive anchors every tap's A
// operand is a 128-row window of ONE contiguous run of rows, so the A operand
// of a tap is the staged run addressed with a row-shifted SWIZZLE_NONE
// K-major shared-memory descriptor (16 B per row).  Anchors with h >= H or
// w >= W are computed and discarded (waste 1 - HW/(HpWp)).
//   * one pipeline stage = (input channel chunk of 16, kd plane): TMA loads the
//     run of R = MB*128 + 2*Wp + 2 rows of the plane for both 8-channel groups
//     and a bulk copy loads the 9 (kh,kw) taps of packed weights;
//   * the MMA warp issues 9 x MB tcgen05.mma (M=128, N=Cout chunk, K=16) per
//     stage into MB accumulators (double-buffered in TMEM across work units);
//   * 4 epilogue warps drain TMEM (tcgen05.ld), add bias, apply ReLU or the
//     previous layer's ReLU mask (dgrad), round to bf16 and store the interior.
// Semantics: conv3d_local ops.py:69-97 (fwd); conv3d_input_grad_local
// ops.py:100-114 == forward of the halo'd output gradient with flipped,
// transposed taps (packed by vm_pack_weights(flip_transpose=1)).
//
// Weight gradient: D[(kd,kh,ci), co] per kw = sum_v x[v + off][ci] * gy[v][co],
// M = 128 rows formed by 16 channel groups of the 9 (kd,kh) row-shifted copies
// of the staged input (MN-major A), N = Cout, K = anchors (MN-major B = gy);
// split-K over anchor ranges, fixed-order reduction (conv3d_param_grads_local,
// ops.py:117-138).
#include <cudaTypedefs.h>

#include "sm100.cuh"
#include "vm_common.cuh"

namespace vm {

using bf16 = __nv_bfloat16;

constexpr int kBoxR = 128;  // TMA box height (rows of 8 bf16 = 16 B)
constexpr int kMaxStages = 6;
constexpr int kSmemBudget = 220 * 1024;
constexpr int kFwdMaxSplit = 16;  // split-K ways of the general forward kernel

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D map over a bf16 slab: (8 channels, Dp*Hp*Wp rows, CG groups, B samples); rows past
// the plane are out of bounds and read as zeros.
static int make_slab_map(CUtensorMap* m, const void* base, int64_t bstride, int CG, int64_t rows,
                         int B, int boxr) {
  auto enc = encode_fn();
  VM_REQUIRE(enc, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  VM_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, VM_E_ALIGN, "slab base not 16B aligned");
  cuuint64_t dims[4] = {8, (cuuint64_t)rows, (cuuint64_t)CG, (cuuint64_t)B};
  cuuint64_t strides[3] = {16, (cuuint64_t)rows * 16, (cuuint64_t)bstride * 2};
  cuuint32_t box[4] = {8, (cuuint32_t)boxr, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  VM_REQUIRE(r == CUDA_SUCCESS, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return VM_OK;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------ weight packing
// Packed forward operand, two layouts chosen by shape (ci = (kc*2 + half)*8 + e):
//  * plain  (k_conv_fwd_tc):    [nchunk][kc][kd][9 taps (kh,kw)][2 K-halves][Nc][8],
//                               co = nchunk*Nc + n;
//  * sweep  (k_conv_fwd_sweep): [kc][9 taps (kh,kw)][2 K-halves][3*Nc][8], row n holds
//                               kd = 2 - n / Nc, co = n % Nc (thin outputs, Nc <= 48);
//  * sweep-kw (k_conv_fwd_sweepkw, Nc = 16): [kc][3 kh][2 K-halves][144][8], row n holds
//                               kd = 2 - n / 48, kw = n % 48 / 16, co = n % 16.
// flip = 1 packs the dgrad operand W'[t'][ci'][co'] = W[26 - t'][co'][ci'] (conv of the
// output gradient).  Both layouts hold the same number of elements.
struct PackGeom {
  int cin, cout;   // of the conv this operand feeds
  int CG, KC;      // input channel groups, chunks of 2 groups
  int Nc, nchunk;  // N per chunk (multiple of 16, <= 256)
  int sweep;       // 1: kd stacked along N (k_conv_fwd_sweep)
};

constexpr int kSweepMaxNc = 48;  // Nc = 48 (16->48 dgrad): 141 -> 91 us vs k_conv_fwd_tc
constexpr uint32_t kSweepMaxWeightBytes = 100 * 1024;
constexpr bool kSweepEnabled = true;
constexpr bool kSweepKw = true;  // Nc = 16: the kd-and-kw-stacked sweep (N = 144)

__host__ __device__ static PackGeom pack_geom(int cin, int cout) {
  PackGeom g;
  g.cin = cin;
  g.cout = cout;
  g.CG = (cin + 7) / 8;
  g.KC = (g.CG + 1) / 2;
  int npad = (cout + 15) / 16 * 16;
  g.nchunk = (npad + 255) / 256;
  g.Nc = ((npad + g.nchunk - 1) / g.nchunk + 15) / 16 * 16;
  const uint32_t wbytes = (uint32_t)g.KC * 9 * 2 * 3 * g.Nc * 16;
  g.sweep = (kSweepEnabled && g.nchunk == 1 && g.Nc <= kSweepMaxNc && wbytes <= kSweepMaxWeightBytes) ? 1 : 0;
  // kd and kw along N (k_conv_fwd_sweepkw) when a plane has >= 2 K chunks: with one chunk the
  // per-plane MMA work (3 x 2 MMAs) is shorter than the kw-recombining drain of the block it
  // frees (16->16 at 128^3: 67 us vs 52 with k_conv_fwd_sweep; 48->16: 93 vs 123 us)
  if (g.sweep && g.Nc == 16 && g.KC >= 2 && kSweepKw) g.sweep = 2;
  return g;
}

// Value of packed element `r` (see PackGeom for the two layouts).
__device__ __forceinline__ float pack_value(const PackGeom& g, int64_t r, const float* __restrict__ w,
                                            int layer_cin, int layer_cout, int flip) {
  const int e = r % 8;
  r /= 8;
  int kd, kh, kw, kc, co, half;
  if (g.sweep == 2) {  // [kc][3 kh][2 halves][144: (kd = 2 - n/48, kw = n%48/16, co = n%16)][8]
    const int n = r % 144;
    r /= 144;
    half = r % 2;
    r /= 2;
    kh = r % 3;
    kc = (int)(r / 3);
    kd = 2 - n / 48;
    kw = (n % 48) / 16;
    co = n % 16;
  } else if (g.sweep) {
    const int n = r % (3 * g.Nc);
    r /= 3 * g.Nc;
    half = r % 2;
    r /= 2;
    const int j = r % 9;
    kc = (int)(r / 9);
    kh = j / 3;
    kw = j % 3;
    kd = 2 - n / g.Nc;
    co = n % g.Nc;
  } else {
    const int n = r % g.Nc;
    r /= g.Nc;
    half = r % 2;
    r /= 2;
    const int j = r % 9;
    r /= 9;
    kd = r % 3;
    r /= 3;
    kc = r % g.KC;
    const int nch = (int)(r / g.KC);
    kh = j / 3;
    kw = j % 3;
    co = nch * g.Nc + n;
  }
  const int t = (kd * 3 + kh) * 3 + kw;
  const int ci = (kc * 2 + half) * 8 + e;
  if (ci >= g.cin || co >= g.cout) return 0.f;
  return !flip ? w[((int64_t)t * layer_cin + ci) * layer_cout + co]
               : w[((int64_t)(26 - t) * layer_cin + co) * layer_cout + ci];
}

__global__ void k_pack_weights(const float* __restrict__ w, bf16* __restrict__ out, PackGeom g,
                               int layer_cin, int layer_cout, int flip) {
  const int64_t total = (int64_t)g.nchunk * g.KC * 27 * 2LL * g.Nc * 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(pack_value(g, i, w, layer_cin, layer_cout, flip));
}

// ------------------------------------------------------------------ forward kernel
struct FwdParams {
  const bf16* x;
  int64_t x_bstride;
  int R;             // staged rows per group per stage (MB*128 + 2*Wp + 2)
  const bf16* wpk;
  const float* bias;
  bf16* y;
  int64_t y_bstride;
  const bf16* mask;
  int64_t m_bstride;
  int B, D, H, W, Hp, Wp;
  int P;             // Hp*Wp
  int64_t anchors;   // D*P (per sample)
  int64_t plane8;    // Dp*P*8 elements per channel group plane
  int CG, KC;        // input groups, chunks
  int Cout, Nc, nchunk;
  int MB, Ralloc, stages;
  int nacc;          // accumulator sets per tile (kd % nacc): independent MMA chains
  int nbuf;          // TMEM buffers across units (2: epilogue overlaps the next unit)
  int mblocks;       // per sample
  int units;
  uint32_t a_bytes;  // per group per stage
  uint32_t b_bytes;  // per stage
  uint32_t stage_bytes;
  uint32_t idesc;
  unsigned flags;
  long long* dbg;  // optional timing probes [gridDim][8]
  uint32_t wp_magic, hp_magic;  // floor(2^32 / d) + 1 for the anchor (w, h) split
  HaloLink hl;     // fused peer-memory depth halo (vm_conv3d_fwd_tc_link)
  // split-K over the 3*KC (kc, kd) stages: unit = (tile unit tu, split ks); split ks writes
  // f32 partials ws[ks][tu][MB][Nc][128], the last split of a tile unit to finish (counter)
  // sums all splits in split order (deterministic) and runs the epilogue
  int ksplit, spk;
  float* ws;
  int* counters;  // [tile units], zero between launches (the last split resets its counter)
  // 1: the ksplit CTAs of a tile unit are one thread-block cluster (cluster rank = split): each
  // drains its f32 partial into its own shared memory (the free stage buffers) and the fix-up
  // reads the other splits' partials over DSMEM — no global round trip, no arrival counters
  int cluster;
};

// MB (tiles per unit) is a template parameter so that the MMA issue loop is straight-line
// code: measured on B200, a runtime-bounded issue loop costs 1.5x in MMA throughput for
// N = 128 (tools/probes/probe_pipe.cu).
// MODE 0: plain; 1: cycle probes (tools/dbg_fwd_probe.py); 2: fused peer-memory halo (p.hl)
template <int MB, int MODE>
__global__ void __launch_bounds__(320, 1)
    k_conv_fwd_tc(const FwdParams p) {
  constexpr bool DBG = MODE == 1, HL = MODE == 2;
  auto clk = []() -> long long { return DBG ? (long long)clock64() : 0LL; };
  const long long t_kstart = clk();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(16) float sbias[1024];  // Cout <= 1024 (zero-padded to 8); wider: L1
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  pdl_wait();
  if (!(p.flags & kFlagPdlLate)) pdl_trigger();
  const int nstage_k = p.KC * 3;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      if (HL) halo_link_wait(p.hl);  // the input's margins, pushed by the neighbours' producers
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int ks = u % p.ksplit, tu = u / p.ksplit;
        const int nch = tu % p.nchunk;
        const int mb = (tu / p.nchunk) % p.mblocks;
        const int b = tu / (p.nchunk * p.mblocks);
        const int64_t a0 = (int64_t)mb * p.MB * 128;
        const int s0 = ks * p.spk, s1 = min(nstage_k, s0 + p.spk);
        for (int s = s0; s < s1; ++s) {
          const int kc = s / 3, kd = s % 3;
          const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
          {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = smem + (size_t)stage * p.stage_bytes;
            uint8_t* sB = sA + 2 * p.a_bytes;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)ng * p.R * 16 + p.b_bytes);
            // one bulk copy per 8-channel group: the run of R consecutive rows of plane kd
            for (int g = 0; g < ng; ++g)
              bulk_load(sA + (size_t)g * p.a_bytes,
                        p.x + b * p.x_bstride + (kc * 2 + g) * p.plane8 + (a0 + (int64_t)kd * p.P) * 8,
                        (uint32_t)p.R * 16, &full[stage]);
            const bf16* src = p.wpk + (((int64_t)nch * p.KC + kc) * 3 + kd) * (p.b_bytes / 2);
            bulk_load(sB, src, p.b_bytes, &full[stage]);
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    if (p.cluster) {  // the epilogue's two cluster barriers (partials in smem; fix-up done)
      cluster_sync();
      cluster_sync();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    long long t_wait_tmem = 0, t_wait_full = 0, t_start = clk();
    int stage = 0;
    uint32_t phase = 0;
    int ab = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      long long tw0 = clk();
      mbar_wait(&tempty[ab], aphase ^ 1);
      t_wait_tmem += clk() - tw0;
      tc_fence_after();
      const int s0 = (u % p.ksplit) * p.spk, s1 = min(nstage_k, s0 + p.spk);
      // accumulator set of tap j = j % nacc (nacc in {1, 2, 3}): consecutive MMAs of a tile go
      // to different sets, so MB * nacc independent chains are in flight (a single chain of the
      // 9 taps of a stage ran at ~100 cycles per N = 128 MMA against a 64-cycle bound)
      const uint32_t setcol = p.nacc > 1 ? (uint32_t)p.Nc : 0u;
      const int nacc = p.nacc;
      for (int s = s0; s < s1; ++s) {
        const int kc = s / 3;
        const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
        long long tf0 = clk();
        mbar_wait(&full[stage], phase);
        t_wait_full += clk() - tf0;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sB = sA + 2 * p.a_bytes;
          const uint32_t lbo_a = ng == 2 ? p.a_bytes : 0;
          // descriptors advance by plain adds on the 16-byte address field
          const uint64_t a0desc = make_sdesc(sA, lbo_a, 128);
          const uint64_t b0desc = make_sdesc(sB, p.Nc * 16, 128);
          // TMEM column of (buffer ab, tile i, set a) = ((ab*MB + i)*nacc + a)*Nc
          const uint32_t d0 = tbase + (uint32_t)(ab * p.MB * p.nacc * p.Nc);
          const uint32_t tstep = (uint32_t)(p.nacc * p.Nc);
          const uint32_t bstep = (uint32_t)(2 * p.Nc * 16) >> 4;
          const bool first = s == s0;  // the unit's first stage overwrites each set once
          const uint32_t wp1 = (uint32_t)p.Wp;
#pragma unroll
          for (int j = 0; j < 9; ++j) {
            const uint64_t bdesc = b0desc + (uint64_t)(j * bstep);
            const uint64_t adesc = a0desc + (uint64_t)((j / 3) * wp1 + (j % 3));
            const int set = nacc == 3 ? j % 3 : (nacc == 2 ? (j & 1) : 0);
            const uint32_t acc = (first && j < nacc) ? 0u : 1u;
            const uint32_t dj = d0 + (uint32_t)set * setcol;
#pragma unroll
            for (int i = 0; i < MB; ++i)
              mma_bf16_ss(dj + (uint32_t)i * tstep, adesc + (uint64_t)(i * 128), bdesc, p.idesc, acc);
          }
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) mma_commit(&tfull[ab]);
      __syncwarp();
      if (++ab == p.nbuf) {
        ab = 0;
        aphase ^= 1;
      }
    }
    if (p.dbg && lane == 0) {
      p.dbg[blockIdx.x * 8 + 0] = clk() - t_start;
      p.dbg[blockIdx.x * 8 + 1] = t_wait_tmem;
      p.dbg[blockIdx.x * 8 + 2] = t_wait_full;
    }
    if (p.cluster) {
      cluster_sync();
      cluster_sync();
    }
  } else {
    // ===================== epilogue (warps 2..9) =====================
    // warp w drains TMEM lane quarter (w & 3) of every other tile (parity (w-2)/4)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const bool bias_smem = p.Cout <= 1024;
    if (!(p.flags & VM_CONV_NOBIAS) && bias_smem)
      for (int c = threadIdx.x - 64; c < min(1024, (p.Cout + 7) / 8 * 8); c += 256)
        sbias[c] = c < p.Cout ? p.bias[c] : 0.f;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    int ab = 0;
    uint32_t aphase = 0;
    long long t_epi_wait = 0;
    const int ng_out = p.Nc / 8;
    const int ng_half = (ng_out + 1) / 2;
    const bool domask = p.flags & VM_CONV_MASK;
    const int et = threadIdx.x - 64;  // 0..255
    __shared__ int s_last;
    // bias, ReLU / mask, zero beyond Cout, bf16 store of 8 channels of one output row.  Kept
    // free of per-element branches: the drain is instruction-bound (8 warps x 8 channels per
    // call), and the per-element bias/bound selects made it ~500 instructions per 16 channels.
    const bool nobias = p.flags & VM_CONV_NOBIAS;
    const bool relu = p.flags & VM_CONV_RELU;
    const bool cout8 = (p.Cout & 7) == 0;
    auto emit = [&](bf16* ybase, int co0, float (&v)[8], const int4& mkv, int64_t orow, int dq) {
      if (!nobias) {
        float bb[8];
        if (bias_smem) {
          const float4 b0 = *reinterpret_cast<const float4*>(&sbias[co0]);
          const float4 b1 = *reinterpret_cast<const float4*>(&sbias[co0 + 4]);
          bb[0] = b0.x, bb[1] = b0.y, bb[2] = b0.z, bb[3] = b0.w, bb[4] = b1.x, bb[5] = b1.y, bb[6] = b1.z, bb[7] = b1.w;
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) bb[e] = co0 + e < p.Cout ? __ldg(p.bias + co0 + e) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] += bb[e];
      }
      if (relu) {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
      }
      if (domask) {
        const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&mkv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(mh[e]);
          v[2 * e] = f.x > 0.f ? v[2 * e] : 0.f;
          v[2 * e + 1] = f.y > 0.f ? v[2 * e + 1] : 0.f;
        }
      }
      if (!cout8) {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = co0 + e < p.Cout ? v[e] : 0.f;
      }
      int4 out;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
      for (int e = 0; e < 4; ++e) oh[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      if (!(DBG && (p.flags & (1u << 9))))  // probe builds: flag bit 9 skips the store
        *reinterpret_cast<int4*>(ybase + (co0 / 8) * p.plane8 + orow * 8) = out;
      // fused depth halo: layer 1 -> the lo neighbour's layer D+1, layer D -> the hi one's layer 0
      if (HL && p.hl.lo && dq == 0)
        *reinterpret_cast<int4*>(p.hl.lo + (ybase - p.y) + (co0 / 8) * p.plane8 + (orow + p.anchors) * 8) = out;
      if (HL && p.hl.hi && dq == p.D - 1)
        *reinterpret_cast<int4*>(p.hl.hi + (ybase - p.y) + (co0 / 8) * p.plane8 + (orow - p.anchors) * 8) = out;
    };
    // output row of anchor a: (w, h) via multiply-high division (divisors are small)
    auto anchor_row = [&](int a, bool& valid, int& dq) -> int64_t {
      uint32_t qa = __umulhi((uint32_t)a, p.wp_magic);
      if (qa * (uint32_t)p.Wp > (uint32_t)a) --qa;
      if ((qa + 1) * (uint32_t)p.Wp <= (uint32_t)a) ++qa;
      const int wq = a - (int)qa * p.Wp;
      uint32_t qh = __umulhi(qa, p.hp_magic);
      if (qh * (uint32_t)p.Hp > qa) --qh;
      if ((qh + 1) * (uint32_t)p.Hp <= qa) ++qh;
      const int hq = (int)qa - (int)qh * p.Hp;
      dq = (int)qh;
      valid = a < p.anchors && wq < p.W && hq < p.H;
      return (int64_t)a + p.P + p.Wp + 1;
    };
    const int ntu = p.units / p.ksplit;
    const long long t_epi0 = clk();
    long long t_fix = 0, t_pub = 0, t_arr = 0, t_drain = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int ks = u % p.ksplit, tu = u / p.ksplit;
      const int nch = tu % p.nchunk;
      const int mb = (tu / p.nchunk) % p.mblocks;
      const int b = tu / (p.nchunk * p.mblocks);
      const int a0 = mb * p.MB * 128;
      const int s0 = ks * p.spk, nst = min(3 * p.KC, s0 + p.spk) - s0;
      const int nsets = nst > 0 ? p.nacc : 0;  // taps rotate over the sets: all of them written
      const bool split = p.ksplit > 1;
      const bf16* mbase = p.mask + b * p.m_bstride;
      bf16* ybase = p.y + b * p.y_bstride;
      long long te0 = clk();
      mbar_wait(&tfull[ab], aphase);
      const long long taw = clk();
      t_epi_wait += taw - te0;
      tc_fence_after();
      // MB = 1: both warp halves drain the single tile, each half its own channel groups
      const int glo = MB == 1 ? (half ? ng_half : 0) : 0, ghi = MB == 1 ? (half ? ng_out : ng_half) : ng_out;
      for (int i = MB == 1 ? 0 : half; i < p.MB; i += MB == 1 ? 1 : 2) {
        if (DBG && (p.flags & (1u << 11))) break;  // probe builds: flag bit 11 skips the drain
        const int row = q * 32 + lane;
        const int a = a0 + i * 128 + row;
        bool valid;
        int dq;
        const int64_t orow = anchor_row(a, valid, dq);
        const uint32_t tcol = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * p.MB + i) * p.nacc * p.Nc);
        // partial layout [ks][tu][tile][row][Nc]: a thread's channels are contiguous (float4 I/O);
        // cluster splits: [tile][row][Nc] in this CTA's shared memory (the stage buffers)
        float* wsp = !split ? nullptr
                     : p.cluster ? reinterpret_cast<float*>(smem) + ((int64_t)i * 128 + row) * p.Nc
                                 : p.ws + ((((int64_t)ks * ntu + tu) * p.MB + i) * 128 + row) * p.Nc;
        for (int g0 = glo; g0 < ghi; g0 += 8) {
          const int gn = min(8, ghi - g0);
          int4 mk[8];
          if (domask && !split) {  // issue the mask loads first (latency overlap)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int co0 = nch * p.Nc + (g0 + j) * 8;
              mk[j] = make_int4(0, 0, 0, 0);
              if (j < gn && valid && co0 < p.Cout)
                mk[j] = __ldg(reinterpret_cast<const int4*>(mbase + (co0 / 8) * p.plane8 + orow * 8));
            }
          }
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            if (j >= gn) break;
            // sum the accumulator sets in fixed order; the set loop is unrolled (a runtime
            // bound made the compiler rotate all 16 sums through moves every iteration)
            float r[16];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              if (a >= nsets) break;
              uint32_t ra[16];
              const uint32_t ca = tcol + (uint32_t)(a * p.Nc + (g0 + j) * 8);
              if (j + 1 < gn) {
                tmem_ld16(ca, ra);
              } else {
                uint32_t r8[8];
                tmem_ld8(ca, r8);
#pragma unroll
                for (int e = 0; e < 8; ++e) ra[e] = r8[e];
#pragma unroll
                for (int e = 8; e < 16; ++e) ra[e] = 0u;
              }
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e) r[e] = a == 0 ? __uint_as_float(ra[e]) : r[e] + __uint_as_float(ra[e]);
            }
            if (split) {  // f32 partial of 8 or 16 channels of this row
              float4* dst = reinterpret_cast<float4*>(wsp + (g0 + j) * 8);
              if (p.cluster) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (e < 2 || j + 1 < gn) dst[e] = make_float4(r[4 * e], r[4 * e + 1], r[4 * e + 2], r[4 * e + 3]);
              } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (e < 2 || j + 1 < gn) __stcg(dst + e, make_float4(r[4 * e], r[4 * e + 1], r[4 * e + 2], r[4 * e + 3]));
              }
              continue;
            }
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              if (j + jj >= gn) break;
              const int co0 = nch * p.Nc + (g0 + j + jj) * 8;
              if (!valid || co0 >= p.Cout) continue;
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = r[jj * 8 + e];
              emit(ybase, co0, v, mk[j + jj], orow, dq);
            }
          }
        }
      }
      t_drain += clk() - taw;
      tc_fence_before();
      mbar_arrive(&tempty[ab]);
      if (++ab == p.nbuf) {
        ab = 0;
        aphase ^= 1;
      }
      if (split) {
        // publish this split's partial, wait for the tile's other splits (all resident: the
        // planner keeps split plans to one wave), then every split finishes its own slice of
        // the tile's rows: the fix-up runs on ksplit CTAs at once instead of the last arriver
        // (one CTA reading every split's partial ran ~49 K cycles for 8 splits of a 512-channel
        // tile: latency-bound)
        const long long tpa = clk();
        if (p.cluster) {
          // every split's partial is in its CTA's shared memory once the cluster barrier
          // completes; the fix-up sums the splits of this CTA's row slice over DSMEM, in split
          // (cluster rank) order, and a second barrier keeps every CTA's shared memory alive
          // until the whole cluster has read it
          cluster_sync();
          t_pub += clk() - tpa;
          t_arr = clk() - t_epi0;
          const long long tfx = clk();
          const int rps = (128 + p.ksplit - 1) / p.ksplit;
          const int rlo = ks * rps, rhi = min(128, rlo + rps);
          const int gvalid = min(ng_out, (p.Cout - nch * p.Nc + 7) / 8);
          const int items = p.MB * (rhi > rlo ? rhi - rlo : 0) * gvalid;
          const uint32_t sbase = smem_u32(smem);
          for (int it = et; it < items; it += 256) {
            const int g = it % gvalid, ri = it / gvalid;
            const int i = ri / (rhi - rlo), row = rlo + ri % (rhi - rlo);
            bool valid;
            int dq;
            const int64_t orow = anchor_row(a0 + i * 128 + row, valid, dq);
            if (!valid) continue;
            const int co0 = nch * p.Nc + g * 8;
            int4 mkv = make_int4(0, 0, 0, 0);
            if (domask) mkv = __ldg(reinterpret_cast<const int4*>(mbase + (co0 / 8) * p.plane8 + orow * 8));
            const uint32_t off = sbase + (uint32_t)((((i * 128 + row) * p.Nc) + g * 8) * 4);
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = 0.f;
            for (int k0 = 0; k0 < p.ksplit; k0 += 4) {  // 4 splits' loads in flight, then the adds
              float4 lo[4], hi[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                if (k0 + j >= p.ksplit) break;
                const uint32_t ra = dsmem_map(off, (uint32_t)(k0 + j));
                lo[j] = dsmem_ld_f4(ra), hi[j] = dsmem_ld_f4(ra + 16);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {  // split order: deterministic
                if (k0 + j >= p.ksplit) break;
                v[0] += lo[j].x, v[1] += lo[j].y, v[2] += lo[j].z, v[3] += lo[j].w;
                v[4] += hi[j].x, v[5] += hi[j].y, v[6] += hi[j].z, v[7] += hi[j].w;
              }
            }
            emit(ybase, co0, v, mkv, orow, dq);
          }
          cluster_sync();
          t_fix += clk() - tfx;
          continue;
        }
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (et == 0) {
          atomicAdd(p.counters + tu, 1);
          const long long tw0 = clock64();
          while (ld_acquire_gpu_i32(p.counters + tu) < p.ksplit) {
            __nanosleep(64);
            if (clock64() - tw0 > 20000000000LL) break;  // never hang the device
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        __threadfence();
        t_pub += clk() - tpa;
        t_arr = clk() - t_epi0;
        const long long tfx = clk();
        // every thread owns (row, channel group) items of this split's row slice: 256 items in
        // flight per CTA, consecutive threads across a row's groups (coalesced partial rows),
        // 4 splits' loads issued per item before the adds (one row per warp at a time was
        // latency-bound: 13 K cycles for the 2-split fix-up of a 128-channel tile)
        const int rps = (128 + p.ksplit - 1) / p.ksplit;
        const int rlo = ks * rps, rhi = min(128, rlo + rps);
        const int gvalid = min(ng_out, (p.Cout - nch * p.Nc + 7) / 8);
        const int items = p.MB * (rhi > rlo ? rhi - rlo : 0) * gvalid;
        for (int it = et; it < items; it += 256) {
          const int g = it % gvalid, ri = it / gvalid;
          const int i = ri / (rhi - rlo), row = rlo + ri % (rhi - rlo);
          bool valid;
          int dq;
          const int64_t orow = anchor_row(a0 + i * 128 + row, valid, dq);
          if (!valid) continue;
          const int co0 = nch * p.Nc + g * 8;
          int4 mkv = make_int4(0, 0, 0, 0);
          if (domask) mkv = __ldg(reinterpret_cast<const int4*>(mbase + (co0 / 8) * p.plane8 + orow * 8));
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = 0.f;
          const float* src0 = p.ws + (((int64_t)tu * p.MB + i) * 128 + row) * p.Nc + g * 8;
          const int64_t kstride = (int64_t)ntu * p.MB * 128 * p.Nc;
          for (int k0 = 0; k0 < p.ksplit; k0 += 4) {
            float4 lo[4], hi[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (k0 + j >= p.ksplit) break;
              const float4* src = reinterpret_cast<const float4*>(src0 + (k0 + j) * kstride);
              lo[j] = __ldcg(src), hi[j] = __ldcg(src + 1);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // split order: deterministic
              if (k0 + j >= p.ksplit) break;
              v[0] += lo[j].x, v[1] += lo[j].y, v[2] += lo[j].z, v[3] += lo[j].w;
              v[4] += hi[j].x, v[5] += hi[j].y, v[6] += hi[j].z, v[7] += hi[j].w;
            }
          }
          emit(ybase, co0, v, mkv, orow, dq);
        }
        // the last split to leave resets both counters for the next launch
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (et == 0 && atomicAdd(p.counters + ntu + tu, 1) == p.ksplit - 1) {
          p.counters[tu] = 0;
          p.counters[ntu + tu] = 0;
        }
        t_fix += clk() - tfx;
      }
    }
    if (p.dbg && threadIdx.x == 64) {
      p.dbg[blockIdx.x * 8 + 3] = t_epi_wait;
      p.dbg[blockIdx.x * 8 + 4] = clk() - t_epi0;
      p.dbg[blockIdx.x * 8 + 5] = t_fix;
      p.dbg[blockIdx.x * 8 + 6] = p.ksplit > 1 ? t_pub : t_drain;
      p.dbg[blockIdx.x * 8 + 7] = p.ksplit > 1 ? t_arr : t_epi0 - t_kstart;
    }
  }
  tc_fence_before();
  if (HL && p.hl.counter) __threadfence();  // every thread's halo pushes, before the CTA counts itself
  __syncthreads();
  if (HL && threadIdx.x == 0) halo_link_signal(p.hl);
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ weight-gradient kernel
// Rows of M: 16 channel groups per M-tile, group g = p*CG + cg with p = kd*3 + kh.
// Each group is staged by one bulk copy as its own run of KS+8 rows (the
// (kd,kh)-shifted input), so consecutive groups sit at a uniform stride (SBO)
// and the kw shift is a 16-byte start-address offset along K.  B = gy rows
// (MN-major, co groups) fetched by ONE 128B-inner TMA box per stage.  A spare
// M slot (when 9*CG is not a multiple of 16) holds a block of ones, so the same
// MMAs also produce the bias gradient sum_v gy[v][co].
struct WgParams {
  const bf16* x;
  int64_t x_bstride;
  int64_t plane8;   // elements per channel-group plane
  int B, D, H, W, Hp, Wp, P;
  int CG, CGo, Cout, Nc;  // CGo: gy channel groups staged per unit (Nc / 8 of one output chunk)
  int nchunk, NcTot;      // output-channel chunks of Nc in this launch (NcTot = nchunk * Nc)
  int KS, RR;       // anchors per stage, staged rows per group (KS + 8)
  int gdelta;       // row misalignment of the gy box start (128B-inner mode)
  int gwide;        // 1: gy map has 128-byte inner boxes
  int MT, mt_per_unit, n_mtgroups;
  int ones_slot;    // absolute M slot of the ones block, -1 if none
  int runs;         // 1: stage one run of KS+2Wp+2 rows per (kd, cg) serving all three kh
                    //    (M slot g' = (kd*CG + cg)*3 + kh, slot stride Wp rows); 0: one copy per slot
  int runs_alloc;   // run slots per stage buffer (runs mode)
  int spk;          // stages per unit (K-split chunk)
  int ksplit;       // K-split chunks per sample
  int kinter;       // 1: stages interleaved over the split CTAs (L2 reuse of the gy rows)
  int stages_total; // per sample
  int units;
  int grid;         // CTAs (a multiple of n_mtgroups); one K partial per CTA
  int stages;       // pipeline depth
  uint32_t a_bytes; // per stage: mt_per_unit*16 slots * RR * 16
  uint32_t g_bytes; // per stage loaded: CGo * RR * 16 (allocated: Nc/8 groups)
  uint32_t stage_bytes;
  uint32_t idesc;
  float* ws;        // [kidx = b*ksplit + ks][MT][3][NcTot][128]
  long long* dbg;   // optional cycle probes [gridDim][8] (vm_debug_set_fwd_probe)
};

// NMT > 0: M-tiles per CTA, NKK > 0: K steps per stage (KS/16), known at compile time so the
// MMA issue is straight-line code (a runtime-bounded issue loop costs 1.5-2x on B200); 0: runtime.
template <int NMT, int NKK>
__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad_tc(const __grid_constant__ CUtensorMap gmap, const WgParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const bool dbg = p.dbg != nullptr;
  const long long t_entry = dbg ? (long long)clock64() : 0;
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull, tempty;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // every unit of this CTA has the same (output chunk, M-tile group) column
  const int ncol = p.n_mtgroups * p.nchunk;
  const int col = blockIdx.x % ncol;
  const int mg_cta = col % p.n_mtgroups, chunk = col / p.n_mtgroups;
  const int mt0 = mg_cta * p.mt_per_unit;
  const int nmt = min(p.mt_per_unit, p.MT - mt0);
  // ones block for the bias gradient, written once into every stage buffer
  // slot geometry: slot i of this CTA's M-tiles sits at (i + slot_shift) * GS bytes
  const int r0 = p.runs ? (16 * mt0) / 3 : 0;
  const int slot_shift = p.runs ? 16 * mt0 - 3 * r0 : 0;
  const uint32_t GS = (uint32_t)(p.runs ? p.Wp : p.RR) * 16;
  if (p.ones_slot >= 0 && p.ones_slot / 16 >= mt0 && p.ones_slot / 16 < mt0 + nmt) {
    const int local = p.ones_slot - mt0 * 16 + slot_shift;
    const uint32_t one2 = 0x3F803F80u;  // two bf16 1.0
    for (int s = 0; s < p.stages; ++s) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(smem + (size_t)s * p.stage_bytes + (size_t)local * GS);
      for (int i = threadIdx.x; i < (p.KS + 8) * 4; i += blockDim.x) dst[i] = one2;
    }
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  pdl_wait();  // dependents launch as this grid's CTAs exit (no early trigger)
  const int ngroups_total = 9 * p.CG;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&gmap);
      long long t_pe = 0;
      int stage = 0;
      uint32_t phase = 0;
      int nvalid = 0;
      const int r_end = min(3 * p.CG - 1, (16 * (mt0 + nmt) - 1) / 3);  // last valid run (runs mode)
      const int Rrun = p.KS + 2 * p.Wp + 2;
      if (p.runs) {
        nvalid = r_end >= r0 ? r_end - r0 + 1 : 0;
      } else {
        for (int i = 0; i < nmt * 16; ++i)
          if (mt0 * 16 + i < ngroups_total) ++nvalid;
      }
      const uint32_t tx = (uint32_t)nvalid * (p.runs ? Rrun : p.RR) * 16 + p.g_bytes;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int ks = (u / ncol) % p.ksplit;
        const int b = u / (ncol * p.ksplit);
        // K stages interleaved over the split CTAs (stage s -> CTA s % ksplit): at any time the
        // CTAs read one contiguous window of rows, and the kd-shifted gy slices (1-2 planes back)
        // were read a few windows earlier by other CTAs: L2 hits instead of DRAM re-reads
        const int s0 = p.kinter ? ks : ks * p.spk, s1 = p.kinter ? p.stages_total : min(p.stages_total, s0 + p.spk);
        const int sstep = p.kinter ? p.ksplit : 1;
        const bf16* xb = p.x + b * p.x_bstride;
        for (int s = s0; s < s1; s += sstep) {
          const int64_t k0 = (int64_t)s * p.KS;
          const long long tw = dbg ? (long long)clock64() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (dbg) t_pe += clock64() - tw;
          uint8_t* sA = smem + (size_t)stage * p.stage_bytes;
          uint8_t* sG = sA + p.a_bytes;
          mbar_arrive_expect_tx(&full[stage], tx);
          const int gr0 = (int)(k0 + p.P + p.Wp + 1);
          if (p.gwide)
            tma_load_4d(sG, &gmap, &full[stage], 0, (gr0 - p.gdelta) >> 3, chunk * p.CGo, b);
          else
            tma_load_4d(sG, &gmap, &full[stage], 0, gr0, chunk * p.CGo, b);
          if (p.runs) {
            for (int r = r0; r <= r_end; ++r) {
              const int kd = r / p.CG, cg = r % p.CG;
              const bf16* src = xb + cg * p.plane8 + (k0 + (int64_t)kd * p.P) * 8;
              bulk_load(sA + (size_t)(r - r0) * 3 * GS, src, (uint32_t)Rrun * 16, &full[stage]);
            }
          } else {
            for (int i = 0; i < nmt * 16; ++i) {
              const int g = mt0 * 16 + i;
              if (g >= ngroups_total) break;
              const int pp = g / p.CG, cg = g % p.CG;
              const int kd = pp / 3, kh = pp % 3;
              const bf16* src = xb + cg * p.plane8 + (k0 + (int64_t)kd * p.P + (int64_t)kh * p.Wp) * 8;
              bulk_load(sA + (size_t)i * p.RR * 16, src, p.RR * 16, &full[stage]);
            }
          }
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (dbg) p.dbg[blockIdx.x * 8 + 5] = t_pe;
    }
  } else if (warp == 1) {
    // All units of this CTA share the M-tile group and cover disjoint K ranges: accumulate
    // them in TMEM and drain once (one partial per CTA instead of one per unit).
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sbo = GS;
    bool started = false;
    const long long t_m0 = dbg ? (long long)clock64() : 0;
    long long t_wf = 0, t_first = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int ks = (u / ncol) % p.ksplit;
      // K stages interleaved over the split CTAs (stage s -> CTA s % ksplit): at any time the
      // CTAs read one contiguous window of rows, and the kd-shifted gy slices (1-2 planes back)
      // were read a few windows earlier by other CTAs: L2 hits instead of DRAM re-reads
      const int s0 = p.kinter ? ks : ks * p.spk, s1 = p.kinter ? p.stages_total : min(p.stages_total, s0 + p.spk);
      const int sstep = p.kinter ? p.ksplit : 1;
      for (int s = s0; s < s1; s += sstep) {
        const long long tw = dbg ? (long long)clock64() : 0;
        mbar_wait(&full[stage], phase);
        if (dbg) {
          const long long dt = clock64() - tw;
          if (!started) t_first = dt; else t_wf += dt;
        }
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sG = sA + p.a_bytes;
          const uint64_t b0desc = make_sdesc(sG + (uint32_t)p.gdelta * 16, 128, (uint32_t)p.RR * 16);
          const uint64_t a0desc = make_sdesc(sA + (uint32_t)slot_shift * GS, 128, sbo);
          const uint32_t mstep = 16 * (GS >> 4);  // 16 slots, in 16-byte units
          const int nkk = NKK > 0 ? NKK : p.KS / 16;
          const uint32_t acc0 = started ? 1u : 0u;
          if (NMT > 0 && NKK > 0) {
#pragma unroll
            for (int kk = 0; kk < (NKK > 0 ? NKK : 1); ++kk) {
              const uint64_t bdesc = b0desc + (uint64_t)(kk * 16);
              const uint32_t acc = kk > 0 ? 1u : acc0;
#pragma unroll
              for (int m = 0; m < (NMT > 0 ? NMT : 1); ++m) {
                const uint64_t adesc = a0desc + (uint64_t)(m * mstep + kk * 16);
                const uint32_t d = tbase + (uint32_t)(m * 3 * p.Nc);
                mma_bf16_ss(d, adesc, bdesc, p.idesc, acc);
                mma_bf16_ss(d + p.Nc, adesc + 1, bdesc, p.idesc, acc);
                mma_bf16_ss(d + 2 * p.Nc, adesc + 2, bdesc, p.idesc, acc);
              }
            }
          } else if (NMT > 0) {
          } else {
#pragma unroll 1
            for (int kk = 0; kk < nkk; ++kk) {
              const uint64_t bdesc = b0desc + (uint64_t)(kk * 16);
              const uint32_t acc = kk > 0 ? 1u : acc0;
#pragma unroll 1
              for (int m = 0; m < nmt; ++m) {
                const uint64_t adesc = a0desc + (uint64_t)(m * mstep + kk * 16);
                const uint32_t d = tbase + (uint32_t)(m * 3 * p.Nc);
                mma_bf16_ss(d, adesc, bdesc, p.idesc, acc);
                mma_bf16_ss(d + p.Nc, adesc + 1, bdesc, p.idesc, acc);
                mma_bf16_ss(d + 2 * p.Nc, adesc + 2, bdesc, p.idesc, acc);
              }
            }
          }
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        started = true;
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (elect_one()) mma_commit(&tfull);
    __syncwarp();
    if (dbg && lane == 0) {
      p.dbg[blockIdx.x * 8 + 0] = t_m0 - t_entry;
      p.dbg[blockIdx.x * 8 + 1] = clock64() - t_m0;
      p.dbg[blockIdx.x * 8 + 2] = t_first;
      p.dbg[blockIdx.x * 8 + 3] = t_wf;
    }
  } else {
    const int q = warp & 3;
    const int kidx = blockIdx.x / ncol;
    mbar_wait(&tfull, 0);
    tc_fence_after();
    const int m_row = q * 32 + lane;
    for (int m = 0; m < nmt; ++m)
      for (int kw = 0; kw < 3; ++kw)
        for (int n0 = 0; n0 < p.Nc; n0 += 16) {
          uint32_t r[16];
          tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((m * 3 + kw) * p.Nc + n0), r);
          tmem_ld_wait();
          float* dst = p.ws + ((((int64_t)kidx * p.MT + mt0 + m) * 3 + kw) * p.NcTot + chunk * p.Nc + n0) * 128 + m_row;
#pragma unroll
          for (int e = 0; e < 16; ++e) dst[e * 128] = __uint_as_float(r[e]);
        }
    (void)tempty;
    if (dbg && threadIdx.x == 64) p.dbg[blockIdx.x * 8 + 4] = clock64() - t_entry;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// Fixed-order reduction of the nk K-split partials ws[k][mt][kw][n][m] (E floats per split)
// and scatter into gw[t][ci][co] (+ gb from the ones slot or from bias partials).
//   KD = false (k_conv_wgrad_tc): n = co, slot g = mt*16 + m/8 -> (kd*3 + kh, cg);
//   KD = true  (k_conv_wgrad_kd): n = kd*Nc + co, slot g = cg*3 + kh.
// A block owns a 32 (m) x 8 (n) tile.  Warp w sums splits k = w, w+8, ... for all 8 n
// (8 independent coalesced 128-byte loads per k), the 8 warp sums are added in warp order
// through shared memory (deterministic), and the tile is written transposed so that 8
// consecutive co (32 bytes) go out together; the old one-warp-per-32-elements version wrote
// 4-byte scattered stores with a Cout stride.  Blocks past the tiles reduce the separate
// bias partials wsb[nsb][CGo*8] when the ones slot does not exist.  ldo: row stride of gw
// (the full Cout when this call covers a chunk of the output channels).
template <bool KD, int NW>  // NW warps per block split the K partials (32 when there are many)
__global__ void __launch_bounds__(NW * 32) k_wgrad_finalize_tiles(const float* __restrict__ ws, float* __restrict__ gw,
                                                             float* __restrict__ gb, int nk, int MT, int Nc, int CG,
                                                             int Cin, int Cout, int ones_slot, int runs,
                                                             const float* __restrict__ wsb, int nsb, int CGo,
                                                             int ldo, int ci_stride) {
  pdl_wait();
  __shared__ float part[NW][8][33];
  const int N = KD ? 3 * Nc : Nc;
  const int n8 = N / 8;
  const int64_t E = (int64_t)MT * 3 * N * 128;
  const int ntiles = MT * 3 * n8 * 4;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if ((int)blockIdx.x >= ntiles) {
    const int co = ((int)blockIdx.x - ntiles) * (NW * 32) + threadIdx.x;
    if (co < Cout && gb) {
      float sb = 0.f;
      for (int sp = 0; sp < nsb; ++sp) sb += wsb[(int64_t)sp * CGo * 8 + co];
      gb[co] = sb;
    }
    return;
  }
  int r = blockIdx.x;
  const int mq = r % 4;
  r /= 4;
  const int nb = r % n8;
  r /= n8;
  const int kw = r % 3;
  const int mt = r / 3;
  {  // a block whose 4 slots hold neither a kernel row nor the ones (bias) slot writes nothing:
     // skip its partial reads (M = 64 / partly filled M-tiles of the thin layers)
    const int g_lo = mt * 16 + mq * 4;
    const bool live = g_lo < (KD ? 3 : 9) * CG || (ones_slot >= g_lo && ones_slot < g_lo + 4);
    if (!live) return;
  }
  const int64_t e0 = (((int64_t)(mt * 3 + kw) * N + nb * 8) * 128) + mq * 32 + lane;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  for (int k = w; k < nk; k += NW) {
    const float* src = ws + (int64_t)k * E + e0;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = src[j * 128];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += v[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[w][j][lane] = acc[j];
  __syncthreads();
  // thread -> (m = mq*32 + mm, n = nb*8 + j): 8 consecutive n per m
  if (threadIdx.x >= 256) return;
  const int j = threadIdx.x & 7, mm = threadIdx.x >> 3;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) s += part[i][j][mm];
  const int m = mq * 32 + mm;
  const int n = nb * 8 + j;
  const int g = mt * 16 + m / 8;
  int kd, co, pp, cgi;
  bool is_w, is_b;
  if (KD) {
    kd = n / Nc;
    co = n % Nc;
    cgi = g / 3;
    pp = kd * 3 + g % 3;
    is_w = g < 3 * CG && cgi * 8 + m % 8 < Cin;
    is_b = g == ones_slot && kw == 0 && kd == 0 && m % 8 == 0;
  } else {
    co = n;
    pp = runs ? ((g / 3) / CG) * 3 + g % 3 : g / CG;
    cgi = runs ? (g / 3) % CG : g % CG;
    is_w = g < 9 * CG && cgi * 8 + m % 8 < Cin;
    is_b = g == ones_slot && kw == 0 && m % 8 == 0;
  }
  if (co >= Cout) return;
  if (is_w) {
    gw[((int64_t)(pp * 3 + kw) * ci_stride + cgi * 8 + m % 8) * ldo + co] = s;
  } else if (is_b && gb) {
    gb[co] = s;
  }
}

// ------------------------------------------------------------------ forward, kd stacked along N
// Thin outputs (Nc <= 48): the three kd taps are stacked along N (N = 3*Nc, rows ordered
// kd = 2, 1, 0) and a CTA sweeps a column of M tiles (MB*128 in-plane anchors) through a
// segment of depth planes.  Input plane i contributes to output planes i-2, i-1, i, whose
// accumulators are consecutive blocks of a TMEM ring (block = ring sequence mod ring), so
// ONE MMA per (tap (kh,kw), K chunk, tile) covers all three kd taps: 9 MMAs of N = 3*Nc per
// input plane instead of 27 of N = Nc, each input row is staged once per column instead of
// three times, and the A operand (the expensive shared-memory read, ~32 cycles per MMA)
// is read a third as often.  The first K step of a plane overwrites the block of output
// plane i (a separate N = Nc MMA with enable_input_d = 0) and accumulates into the other
// two; a block whose three contributions are issued is committed, drained (bias, ReLU /
// mask, bf16) and handed back.  At the ring's end an MMA is split in two.  Weights stay
// resident in shared memory.  (Pre-filling blocks with the bias by tcgen05.st instead
// serialises the epilogue against in-flight MMAs: 5x slower on B200.)
struct SwParams {
  const bf16* x;
  int64_t x_bstride;
  const bf16* wpk;  // [KC][9][2][3*Nc][8], row n: kd = 2 - n / Nc, co = n % Nc
  const float* bias;
  bf16* y;
  int64_t y_bstride;
  const bf16* mask;
  int64_t m_bstride;
  int D, H, W, Hp, Wp, P;
  int64_t plane8;
  int CG, KC, Cout, Nc;
  int MB;          // M tiles per column (independent accumulator chains: >= 3 hide MMA latency)
  int R;           // staged rows per group per stage = MB*128 + 2*Wp + 2
  int ncol, S, nseg, units;
  int ring;        // TMEM blocks (of Nc columns) per tile
  int stages;
  uint32_t a_bytes, stage_bytes, w_bytes;
  uint32_t idesc1, idesc2, idesc3;
  unsigned flags;
  long long* dbg;  // optional cycle probes [gridDim][8] (vm_debug_set_fwd_probe)
  int xmode;       // experiment: 1 = skip the TMEM drain (wrong results)
  HaloLink hl;     // fused peer-memory depth halo (vm_conv3d_fwd_tc_link)
};
constexpr int kSwMaxRing = 32;
constexpr int kSwMaxStages = 8;

// Warps: 0 producer, 1 and 10 MMA issuers (tiles t = 0, 2, .. and 1, 3, ..: a single issuing
// thread's per-plane bookkeeping otherwise leaves the tensor core idle), 2..9 epilogue.
// NG = Nc/8 channel groups; MODE 0: plain, 1: cycle probes (tools/dbg_sweep_probe.py),
// 2: fused peer-memory halo (p.hl)
// MMA-issuing warps per CTA: one per tile for 16-channel outputs at MB = 4 (warps 1, 10, 11,
// 12; the per-plane bookkeeping of each warp then covers 10 MMAs: measured one warp 61 us,
// two 52 us at 16->16, 128^3), else two (one: MB = 1)
template <int MB, int NG>
constexpr int sweep_mma_warps() {
  return (MB == 4 && NG == 2) ? 4 : (MB >= 2 ? 2 : 1);
}
// epilogue warps (two per TMEM lane quarter; the kernel supports 16: measured no faster for
// 16-channel outputs at MB = 4: fwd 47.4 -> 48.2 us, dgrad 53.2 -> 52.9 us at 128^3)
template <int MB, int NG>
constexpr int sweep_epi_warps() {
  return 8;
}
template <int MB, int NG>
constexpr int sweep_threads() {
  return 32 * (1 + sweep_epi_warps<MB, NG>() + sweep_mma_warps<MB, NG>());
}
template <int MB, int MODE, int NG>
__global__ void __launch_bounds__(sweep_threads<MB, NG>(), 1)
    k_conv_fwd_sweep(const SwParams p) {
  constexpr bool DBG = MODE == 1, HL = MODE == 2;
  auto clk = []() -> long long { return DBG ? (long long)clock64() : 0LL; };
  constexpr int NW = sweep_mma_warps<MB, NG>();  // MMA-issuing warps
  constexpr int EW = sweep_epi_warps<MB, NG>();  // epilogue warps (2 .. EW+1)
  constexpr int NH = EW / 4;                     // epilogue warps per TMEM lane quarter
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kSwMaxStages], empty[kSwMaxStages], tfull[kSwMaxRing], tempty[kSwMaxRing], wbar;
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float sbias[kSweepMaxNc];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint8_t* sW = smem;
  uint8_t* sStage = smem + p.w_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    for (int r = 0; r < p.ring; ++r) {
      mbar_init(&tfull[r], NW);
      mbar_init(&tempty[r], 32 * EW);
    }
    mbar_init(&wbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  pdl_wait();
  if (!(p.flags & kFlagPdlLate)) pdl_trigger();

  if (warp == 0) {
    // ===================== producer: resident weights, then one stage per (plane, K chunk)
    if (elect_one()) {
      mbar_arrive_expect_tx(&wbar, p.w_bytes);
      bulk_load(sW, p.wpk, p.w_bytes, &wbar);
      if (HL) halo_link_wait(p.hl);  // the input's margins, pushed by the neighbours' producers
      int stage = 0;
      uint32_t phase = 0;
      long long t_pw = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int col = u % p.ncol;
        const int seg = (u / p.ncol) % p.nseg;
        const int b = u / (p.ncol * p.nseg);
        const int o0 = seg * p.S, o1 = min(p.D, o0 + p.S);
        const int64_t c0 = (int64_t)col * p.MB * 128;
        const bf16* xb = p.x + b * p.x_bstride;
        for (int i = o0; i < o1 + 2; ++i) {
          for (int kc = 0; kc < p.KC; ++kc) {
            const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
            const long long tw = clk();
            mbar_wait(&empty[stage], phase ^ 1);
            t_pw += clk() - tw;
            uint8_t* sA = sStage + (size_t)stage * p.stage_bytes;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)ng * p.R * 16);
            for (int g = 0; g < ng; ++g)
              bulk_load(sA + (size_t)g * p.a_bytes, xb + (kc * 2 + g) * p.plane8 + ((int64_t)i * p.P + c0) * 8,
                        (uint32_t)p.R * 16, &full[stage]);
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      if (p.dbg) p.dbg[blockIdx.x * 8 + 7] = t_pw;
    }
  } else if (warp == 1 || warp >= 2 + EW) {
    // ===================== MMA issuers
    const int mw = warp == 1 ? 0 : warp - (1 + EW);
    if (mw < NW) {  // (MB = 1: warp 10 idles)
    const long long t0 = clk();
    long long t_te = 0, t_fu = 0, t_is = 0;
    mbar_wait(&wbar, 0);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t nstart = 0;    // ring sequence of the unit's first block (plane o0 - 2)
    uint32_t acquired = 0;  // ring sequences whose block has been re-armed and taken
    uint32_t acq_slot = 0, acq_phase = 0;  // acquired % ring, (acquired / ring) & 1
    uint32_t pos = 0;                      // n % ring (incremental: no divisions per plane)
    const uint32_t wblk = (uint32_t)(2 * 3 * p.Nc * 16);  // bytes per (kc, tap) weight block
    const uint32_t sWa = smem_u32(sW);
    const uint32_t tstride = (uint32_t)(p.ring * p.Nc);   // TMEM columns per tile ring
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int seg = (u / p.ncol) % p.nseg;
      const int o0 = seg * p.S, o1 = min(p.D, o0 + p.S);
      const int nin = o1 - o0 + 2;
      for (int k = 0; k < nin; ++k) {
        const uint32_t n = nstart + (uint32_t)k;
        const long long ta = clk();
        while (acquired <= n + 2) {
          mbar_wait(&tempty[acq_slot], acq_phase);
          ++acquired;
          if (++acq_slot == (uint32_t)p.ring) {
            acq_slot = 0;
            acq_phase ^= 1u;
          }
        }
        t_te += clk() - ta;
        tc_fence_after();
        // Per-plane issue lists, so the issue loop is descriptor adds only (a single thread
        // feeds the tensor core; per-MMA integer work shows up directly as MMA time).
        // Normal K step: blocks pos..pos+2 <- B rows [0, 3Nc), split at the ring's end.
        // First K step: blocks pos..pos+1 accumulate, block pos+2 (plane i) is overwritten.
        const uint32_t ring = (uint32_t)p.ring, Nc = (uint32_t)p.Nc;
        uint32_t nd[2], nid[2], nb[2], fd[3], fid[3], fb[3], facc[3];
        int nn, nf;
        if (pos + 3 <= ring) {
          nn = 1;
          nd[0] = pos * Nc, nid[0] = p.idesc3, nb[0] = 0;
          nd[1] = 0, nid[1] = 0, nb[1] = 0;
        } else if (pos + 2 == ring) {
          nn = 2;
          nd[0] = pos * Nc, nid[0] = p.idesc2, nb[0] = 0;
          nd[1] = 0, nid[1] = p.idesc1, nb[1] = 2 * Nc;
        } else {
          nn = 2;
          nd[0] = pos * Nc, nid[0] = p.idesc1, nb[0] = 0;
          nd[1] = 0, nid[1] = p.idesc2, nb[1] = Nc;
        }
        if (pos + 2 < ring) {  // (pos, pos+1) contiguous
          nf = 2;
          fd[0] = pos * Nc, fid[0] = p.idesc2, fb[0] = 0, facc[0] = 1;
          fd[1] = (pos + 2) * Nc, fid[1] = p.idesc1, fb[1] = 2 * Nc, facc[1] = 0;
          fd[2] = 0, fid[2] = 0, fb[2] = 0, facc[2] = 0;
        } else if (pos + 2 == ring) {
          nf = 2;
          fd[0] = pos * Nc, fid[0] = p.idesc2, fb[0] = 0, facc[0] = 1;
          fd[1] = 0, fid[1] = p.idesc1, fb[1] = 2 * Nc, facc[1] = 0;
          fd[2] = 0, fid[2] = 0, fb[2] = 0, facc[2] = 0;
        } else {
          nf = 3;
          fd[0] = pos * Nc, fid[0] = p.idesc1, fb[0] = 0, facc[0] = 1;
          fd[1] = 0, fid[1] = p.idesc1, fb[1] = Nc, facc[1] = 1;
          fd[2] = Nc, fid[2] = p.idesc1, fb[2] = 2 * Nc, facc[2] = 0;
        }
        for (int kc = 0; kc < p.KC; ++kc) {
          const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
          const long long tf = clk();
          mbar_wait(&full[stage], phase);
          const long long tf1 = clk();
          t_fu += tf1 - tf;
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sA = smem_u32(sStage + (size_t)stage * p.stage_bytes);
            const uint64_t a0desc = make_sdesc(sA, ng == 2 ? p.a_bytes : 0, 128);
            const uint64_t b0desc = make_sdesc(sWa + (uint32_t)kc * 9 * wblk, (uint32_t)(3 * p.Nc * 16), 128);
            const uint32_t wp1 = (uint32_t)p.Wp, wstep = wblk >> 4;
            if (pos + 3 <= ring) {
              // common case, straight-line: blocks pos..pos+2 contiguous
              const uint32_t dpos = tbase + pos * Nc;
              const uint32_t id1 = p.idesc1, id2 = p.idesc2, id3 = p.idesc3;
#pragma unroll
              for (int j = 0; j < 9; ++j) {
                const uint64_t bdesc = b0desc + (uint64_t)(j * wstep);
                const uint64_t adesc = a0desc + (uint64_t)((j / 3) * wp1 + (j % 3));
                // every block arrives zeroed from the epilogue: all MMAs accumulate
#pragma unroll
                for (int tt = 0; tt < (MB + NW - 1) / NW; ++tt) {
                  const int t = mw + tt * NW;
                  if (t >= MB) break;
                  mma_bf16_ss(dpos + t * tstride, adesc + (uint64_t)(t * 128), bdesc, id3, 1u);
                }
              }
            } else {
#pragma unroll 1
            for (int j = 0; j < 9; ++j) {
              const uint64_t bdesc = b0desc + (uint64_t)(j * wstep);
              const uint64_t adesc = a0desc + (uint64_t)((j / 3) * wp1 + (j % 3));
              if (nn == 1) {
#pragma unroll
                for (int tt = 0; tt < (MB + NW - 1) / NW; ++tt) {
                  const int t = mw + tt * NW;
                  if (t >= MB) break;
                  mma_bf16_ss(tbase + t * tstride + nd[0], adesc + (uint64_t)(t * 128), bdesc, nid[0], 1u);
                }
              } else {
#pragma unroll
                for (int tt = 0; tt < (MB + NW - 1) / NW; ++tt) {
                  const int t = mw + tt * NW;
                  if (t >= MB) break;
                  mma_bf16_ss(tbase + t * tstride + nd[0], adesc + (uint64_t)(t * 128), bdesc + nb[0], nid[0], 1u);
                  mma_bf16_ss(tbase + t * tstride + nd[1], adesc + (uint64_t)(t * 128), bdesc + nb[1], nid[1], 1u);
                }
              }
            }
            }  // ring-end planes
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          t_is += clk() - tf1;
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        // block n has received all three contributions (planes below o0 are scratch)
        const uint32_t p1 = pos + 1 == (uint32_t)p.ring ? 0u : pos + 1;
        if (elect_one()) {
          mma_commit(&tfull[pos]);
          if (k == nin - 1) {
            mma_commit(&tfull[p1]);
            mma_commit(&tfull[p1 + 1 == (uint32_t)p.ring ? 0u : p1 + 1]);
          }
        }
        __syncwarp();
        pos = p1;
      }
      nstart += (uint32_t)(nin + 2);
      pos += 2;  // the unit's two trailing blocks
      if (pos >= (uint32_t)p.ring) pos -= (uint32_t)p.ring;
    }
    if (p.dbg && lane == 0 && mw == 0) {
      p.dbg[blockIdx.x * 8 + 0] = clk() - t0;
      p.dbg[blockIdx.x * 8 + 1] = t_te;
      p.dbg[blockIdx.x * 8 + 2] = t_fu;
      p.dbg[blockIdx.x * 8 + 3] = t_is;
    }
    }
  } else {
    // ===================== epilogue (warps 2..9): TMEM lane quarter q, half h
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    // tiles t = h, h+NH, ... of every block (MB = 1: both halves share the tile, split by group)
    constexpr int TPT = MB == 1 ? 1 : (MB + NH - 1) / NH;  // tiles per thread (max)
    // channel groups per thread: compile-time, so the TMEM, mask and prefetch arrays hold
    // exactly the groups this layer has (sized for Nc = 48 they spilled at MB = 3, 4)
    constexpr int GPT = MB == 1 ? (NG + 1) / 2 : NG;
    constexpr int ngrp = NG;
    const int g_lo = MB == 1 ? h : 0, g_step = MB == 1 ? 2 : 1;  // channel groups of this thread
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
    const bool nobias = p.flags & VM_CONV_NOBIAS;
    // every ring block starts at zero and is re-zeroed when drained (tcgen05.st), so all MMAs
    // accumulate (no overwrite split of the first K step: one MMA fewer per tile and plane)
    auto zero_block = [&](uint32_t r) {
      const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const int t = MB == 1 ? 0 : h + NH * k;
        if (t >= MB) break;
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi) {
          const int g = g_lo + gi * g_step;
          if (g < ngrp) tmem_st8(lane_base + (uint32_t)((t * p.ring + (int)r) * p.Nc + g * 8), z);
        }
      }
    };
    for (int r = 0; r < p.ring; ++r) zero_block((uint32_t)r);
    tmem_st_wait();
    tc_fence_before();
    for (int r = 0; r < p.ring; ++r) mbar_arrive(&tempty[r]);
    for (int c = threadIdx.x - 64; c < p.Nc; c += 32 * EW) sbias[c] = (!nobias && c < p.Cout) ? p.bias[c] : 0.f;
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
    uint32_t n = 0;
    uint32_t r = 0, rphase = 0;  // n % ring, (n / ring) & 1
    const long long e0 = clk();
    long long e_w = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int col = u % p.ncol;
      const int seg = (u / p.ncol) % p.nseg;
      const int b = u / (p.ncol * p.nseg);
      const int o0 = seg * p.S, o1 = min(p.D, o0 + p.S);
      const int L = o1 - o0 + 4;
      bool valid[TPT];
      int64_t orow0[TPT];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const int t = MB == 1 ? 0 : h + NH * k;
        const int ra = col * MB * 128 + t * 128 + q * 32 + lane;  // in-plane anchor
        const int hq = ra / p.Wp, wq = ra % p.Wp;
        valid[k] = t < MB && ra < p.P && hq < p.H && wq < p.W;
        orow0[k] = (int64_t)ra + p.P + p.Wp + 1;
      }
      bf16* yb = p.y + b * p.y_bstride;
      const bf16* mb = p.mask + b * p.m_bstride;
      int4 mkn[TPT][GPT];
#pragma unroll
      for (int k = 0; k < TPT; ++k)
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi) mkn[k][gi] = make_int4(0, 0, 0, 0);
      for (int rel = 0; rel < L; ++rel, ++n) {
        const int o = o0 + rel - 2;
        const bool live = o >= o0 && o < o1 && !(p.xmode & 1);  // warp-uniform (tcgen05.ld is .aligned)
        // dgrad: the ReLU mask of the NEXT plane is fetched one plane ahead (mkn), so its HBM
        // latency overlaps this plane's TMEM drain instead of sitting in front of it
        int4 mk[TPT][GPT];
        if (p.flags & VM_CONV_MASK) {
#pragma unroll
          for (int k = 0; k < TPT; ++k)
#pragma unroll
            for (int gi = 0; gi < GPT; ++gi) {
              mk[k][gi] = mkn[k][gi];
              const int g = g_lo + gi * g_step;
              const int on = o + 1;
              mkn[k][gi] = make_int4(0, 0, 0, 0);
              if (on >= o0 && on < o1 && valid[k] && g < ngrp && g * 8 < p.Cout)
                mkn[k][gi] = __ldg(reinterpret_cast<const int4*>(mb + g * p.plane8 + orow0[k] * 8 +
                                                                 (int64_t)on * p.P * 8));
            }
        }
        const long long tw = clk();
        mbar_wait(&tfull[r], rphase);
        e_w += clk() - tw;
        tc_fence_after();
        if (live) {
#pragma unroll
          for (int k = 0; k < TPT; ++k) {
            const int t = MB == 1 ? 0 : h + NH * k;
            if (t >= MB) break;
            const int64_t orow = orow0[k] + (int64_t)o * p.P;
            const uint32_t tcol = lane_base + (uint32_t)((t * p.ring + (int)r) * p.Nc);
            // every group of this tile in flight before one wait
            uint32_t rr[GPT][8];
#pragma unroll
            for (int gi = 0; gi < GPT; ++gi) {
              const int g = g_lo + gi * g_step;
              if (g < ngrp && g * 8 < p.Cout) tmem_ld8(tcol + (uint32_t)(g * 8), rr[gi]);
            }
            tmem_ld_wait();
#pragma unroll
            for (int gi = 0; gi < GPT; ++gi) {
              const int g = g_lo + gi * g_step;
              if (g >= ngrp || g * 8 >= p.Cout) break;
              const float4 b0 = *reinterpret_cast<const float4*>(&sbias[g * 8]);
              const float4 b1 = *reinterpret_cast<const float4*>(&sbias[g * 8 + 4]);
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(rr[gi][e]) + bb[e];
              if (p.flags & VM_CONV_MASK) {
                const uint32_t* mw = reinterpret_cast<const uint32_t*>(&mk[k][gi]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  v[2 * e] = (int16_t)(mw[e] & 0xFFFFu) > 0 ? v[2 * e] : 0.f;
                  v[2 * e + 1] = (int16_t)(mw[e] >> 16) > 0 ? v[2 * e + 1] : 0.f;
                }
              }
              int4 out;
              uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
              if (p.flags & VM_CONV_RELU) {
#pragma unroll
                for (int e = 0; e < 4; ++e) ow[e] = pack_bf16x2_relu(v[2 * e], v[2 * e + 1]);
              } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) ow[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
              }
              if (valid[k]) {
                *reinterpret_cast<int4*>(yb + g * p.plane8 + orow * 8) = out;
                // fused depth halo: layer 1 -> lo neighbour's layer D+1, layer D -> hi's layer 0
                if (HL && p.hl.lo && o == 0)
                  *reinterpret_cast<int4*>(p.hl.lo + (yb - p.y) + g * p.plane8 + (orow + (int64_t)p.D * p.P) * 8) = out;
                if (HL && p.hl.hi && o == p.D - 1)
                  *reinterpret_cast<int4*>(p.hl.hi + (yb - p.y) + g * p.plane8 + (orow - (int64_t)p.D * p.P) * 8) = out;
              }
            }
          }
        }
        zero_block(r);  // (after this block's loads completed: tmem_ld_wait above, or no loads)
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&tempty[r]);
        if (++r == (uint32_t)p.ring) {
          r = 0;
          rphase ^= 1u;
        }
      }
    }
    if (p.dbg && threadIdx.x == 64) {
      p.dbg[blockIdx.x * 8 + 4] = clk() - e0;
      p.dbg[blockIdx.x * 8 + 5] = e_w;
      p.dbg[blockIdx.x * 8 + 6] = (long long)n;
    }
  }
  tc_fence_before();
  if (HL && p.hl.counter) __threadfence();  // every thread's halo pushes, before the CTA counts itself
  __syncthreads();
  if (HL && threadIdx.x == 0) halo_link_signal(p.hl);
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ forward / dgrad, Nc = 16, kd AND kw along N
// k_conv_fwd_sweep with the kw taps moved from the A side to the B side as well: B rows =
// (kd = 2, 1, 0) x (kw = 0..2) x 16 output channels, N = 144, so one MMA per (kh, K chunk)
// covers 9 taps (3 per input plane and K chunk instead of 9, the A tile read once per 144
// outputs instead of per 48: the SS-mode A-operand read no longer bounds the MMA).  The kw
// taps are recombined in the epilogue: the D row of input anchor a holds its kw contribution
// to output anchor a - kw, so out[j] = D0[j] + D1[j+1] + D2[j+2] (lane shuffles, and 2 rows
// through shared memory across TMEM lane quarters).  Tiles advance by 126 anchors (the last
// two rows of a 128-row tile only feed outputs of the next tile).  A drained ring block is
// zeroed by the epilogue (tcgen05.st), so every MMA accumulates (no overwrite split).
// TMEM: MB tiles x ring blocks x 48 columns (kw-block width).
constexpr int kKwTile = 126;
// warps: 0 TMA producer, 1-2 MMA issuers (tile 0 / 1), 3-18 epilogue: 4 per TMEM lane quarter,
// one (tile, channel group) slot each (the drain is latency-bound: 16 warps, 4 per SMSP)
constexpr int kKwThreads = 19 * 32;
template <int MB, int MODE>
__global__ void __launch_bounds__(kKwThreads, 1)
    k_conv_fwd_sweepkw(const SwParams p) {
  constexpr bool DBG = MODE == 1, HL = MODE == 2;
  auto clk = []() -> long long { return DBG ? (long long)clock64() : 0LL; };
  constexpr int NW = MB >= 2 ? 2 : 1;  // MMA-issuing warps
  constexpr int BW = 48;               // TMEM columns per ring block: 3 kw x 16 co
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kSwMaxStages], empty[kSwMaxStages], tfull[kSwMaxRing], tempty[kSwMaxRing], wbar;
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float sbias[16];
  // row exchange across TMEM lane quarters: [slot][parity][quarter][lane0 kw1, lane0 kw2, lane1 kw2][8]
  __shared__ __align__(16) float xch[4][2][4][3][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint8_t* sW = smem;
  uint8_t* sStage = smem + p.w_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    for (int r = 0; r < p.ring; ++r) {
      mbar_init(&tfull[r], NW);
      mbar_init(&tempty[r], 512);
    }
    mbar_init(&wbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  pdl_wait();
  if (!(p.flags & kFlagPdlLate)) pdl_trigger();

  if (warp == 0) {
    // ===================== producer: resident weights, then one stage per (plane, K chunk)
    if (elect_one()) {
      mbar_arrive_expect_tx(&wbar, p.w_bytes);
      bulk_load(sW, p.wpk, p.w_bytes, &wbar);
      if (HL) halo_link_wait(p.hl);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int col = u % p.ncol;
        const int seg = (u / p.ncol) % p.nseg;
        const int b = u / (p.ncol * p.nseg);
        const int o0 = seg * p.S, o1 = min(p.D, o0 + p.S);
        const int64_t c0 = (int64_t)col * MB * kKwTile;
        const bf16* xb = p.x + b * p.x_bstride;
        for (int i = o0; i < o1 + 2; ++i) {
          for (int kc = 0; kc < p.KC; ++kc) {
            const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = sStage + (size_t)stage * p.stage_bytes;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)ng * p.R * 16);
            for (int g = 0; g < ng; ++g)
              bulk_load(sA + (size_t)g * p.a_bytes, xb + (kc * 2 + g) * p.plane8 + ((int64_t)i * p.P + c0) * 8,
                        (uint32_t)p.R * 16, &full[stage]);
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ===================== MMA issuers (warp 1: tile 0, warp 2: tile 1)
    const int mw = warp - 1;
    if (mw < NW) {
      const long long t0 = clk();
      long long t_te = 0, t_fu = 0, t_is = 0;
      mbar_wait(&wbar, 0);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t nstart = 0, acquired = 0, acq_slot = 0, acq_phase = 0, pos = 0;
      const uint32_t wblk = (uint32_t)(2 * 144 * 16);  // bytes per (kc, kh) weight block
      const uint32_t sWa = smem_u32(sW);
      const uint32_t ring = (uint32_t)p.ring;
      const uint32_t tcol0 = tbase + (uint32_t)(mw * p.ring * BW);  // this warp's tile
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int seg = (u / p.ncol) % p.nseg;
        const int o0 = seg * p.S, o1 = min(p.D, o0 + p.S);
        const int nin = o1 - o0 + 2;
        for (int k = 0; k < nin; ++k) {
          const uint32_t n = nstart + (uint32_t)k;
          const long long ta = clk();
          while (acquired <= n + 2) {
            mbar_wait(&tempty[acq_slot], acq_phase);
            ++acquired;
            if (++acq_slot == ring) {
              acq_slot = 0;
              acq_phase ^= 1u;
            }
          }
          t_te += clk() - ta;
          tc_fence_after();
          // blocks pos, pos+1, pos+2 (output planes i-2, i-1, i) <- B rows [0,48), [48,96), [96,144)
          const uint32_t d0 = tcol0 + pos * BW;
          const int wrap = pos + 3 <= ring ? 0 : (pos + 2 == ring ? 2 : 1);  // blocks before the ring end
          for (int kc = 0; kc < p.KC; ++kc) {
            const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
            const long long tf = clk();
            mbar_wait(&full[stage], phase);
            const long long tf1 = clk();
            t_fu += tf1 - tf;
            tc_fence_after();
            if (elect_one()) {
              const uint32_t sA = smem_u32(sStage + (size_t)stage * p.stage_bytes);
              const uint64_t a0desc = make_sdesc(sA, ng == 2 ? p.a_bytes : 0, 128) + (uint64_t)(mw * kKwTile);
              const uint64_t b0desc = make_sdesc(sWa + (uint32_t)kc * 3 * wblk, 144 * 16, 128);
              const uint32_t wp1 = (uint32_t)p.Wp, wstep = wblk >> 4;
              if (wrap == 0) {
#pragma unroll
                for (int kh = 0; kh < 3; ++kh)
                  mma_bf16_ss(d0, a0desc + (uint64_t)(kh * wp1), b0desc + (uint64_t)(kh * wstep), p.idesc3, 1u);
              } else if (wrap == 2) {  // blocks pos, pos+1 | 0
#pragma unroll
                for (int kh = 0; kh < 3; ++kh) {
                  const uint64_t ad = a0desc + (uint64_t)(kh * wp1), bd = b0desc + (uint64_t)(kh * wstep);
                  mma_bf16_ss(d0, ad, bd, p.idesc2, 1u);
                  mma_bf16_ss(tcol0, ad, bd + 96, p.idesc1, 1u);
                }
              } else {  // block pos | 0, 1
#pragma unroll
                for (int kh = 0; kh < 3; ++kh) {
                  const uint64_t ad = a0desc + (uint64_t)(kh * wp1), bd = b0desc + (uint64_t)(kh * wstep);
                  mma_bf16_ss(d0, ad, bd, p.idesc1, 1u);
                  mma_bf16_ss(tcol0, ad, bd + 48, p.idesc2, 1u);
                }
              }
              mma_commit(&empty[stage]);
            }
            __syncwarp();
            t_is += clk() - tf1;
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          const uint32_t p1 = pos + 1 == ring ? 0u : pos + 1;
          if (elect_one()) {
            mma_commit(&tfull[pos]);
            if (k == nin - 1) {
              mma_commit(&tfull[p1]);
              mma_commit(&tfull[p1 + 1 == ring ? 0u : p1 + 1]);
            }
          }
          __syncwarp();
          pos = p1;
        }
        nstart += (uint32_t)(nin + 2);
        pos += 2;
        if (pos >= ring) pos -= ring;
      }
      if (DBG && lane == 0 && mw == 0) {
        p.dbg[blockIdx.x * 8 + 0] = clk() - t0;
        p.dbg[blockIdx.x * 8 + 1] = t_te;
        p.dbg[blockIdx.x * 8 + 2] = t_fu;
        p.dbg[blockIdx.x * 8 + 3] = t_is;
      }
    }
  } else {
    // ===================== epilogue (warps 3..18): TMEM lane quarter q, slot hh = (tile, group)
    const int q = warp & 3;
    const int hh = (warp - 3) >> 2;
    constexpr int GPT = 1;
    const int t = hh >> 1;  // MB = 1: slots 2-3 have no tile (they only hand blocks back)
    const int g_lo = hh & 1;
    const bool has_tile = t < MB;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((has_tile ? t : 0) * p.ring * BW);
    const bool nobias = p.flags & VM_CONV_NOBIAS;
    // every ring block starts at zero (MMAs only accumulate), then is handed to the MMA warps
    {
      const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (has_tile) {
        for (int r = 0; r < p.ring; ++r)
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) tmem_st8(lane_base + (uint32_t)(r * BW + kw * 16 + g_lo * 8), z);
      }
      tmem_st_wait();
      tc_fence_before();
      for (int r = 0; r < p.ring; ++r) mbar_arrive(&tempty[r]);
    }
    for (int c = threadIdx.x - 96; c < 16; c += 512) sbias[c] = (!nobias && c < p.Cout) ? p.bias[c] : 0.f;
    asm volatile("bar.sync 1, 512;" ::: "memory");
    const int m = q * 32 + lane;  // TMEM row of this thread
    uint32_t n = 0, r = 0, rphase = 0;
    const long long e0 = clk();
    long long e_w = 0, e_ld = 0, e_x = 0, e_m = 0, e_sw = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int col = u % p.ncol;
      const int seg = (u / p.ncol) % p.nseg;
      const int b = u / (p.ncol * p.nseg);
      const int o0 = seg * p.S, o1 = min(p.D, o0 + p.S);
      const int L = o1 - o0 + 4;
      const int ra = col * MB * kKwTile + t * kKwTile + m;  // output in-plane anchor of row m
      const int hq = ra / p.Wp, wq = ra % p.Wp;
      const bool valid = has_tile && m < kKwTile && ra < p.P && hq < p.H && wq < p.W;
      const int64_t orow0 = (int64_t)ra + p.P + p.Wp + 1;
      bf16* yb = p.y + b * p.y_bstride;
      const bf16* mb = p.mask + b * p.m_bstride;
      int4 mkn[GPT];
#pragma unroll
      for (int gi = 0; gi < GPT; ++gi) mkn[gi] = make_int4(0, 0, 0, 0);
      for (int rel = 0; rel < L; ++rel, ++n) {
        const int o = o0 + rel - 2;
        const bool live = o >= o0 && o < o1;
        int4 mk[GPT];
        if (p.flags & VM_CONV_MASK) {
#pragma unroll
          for (int gi = 0; gi < GPT; ++gi) {
            mk[gi] = mkn[gi];
            const int g = g_lo + gi;
            const int on = o + 1;
            mkn[gi] = make_int4(0, 0, 0, 0);
            if (on >= o0 && on < o1 && valid && g * 8 < p.Cout)
              mkn[gi] = __ldg(reinterpret_cast<const int4*>(mb + g * p.plane8 + orow0 * 8 + (int64_t)on * p.P * 8));
          }
        }
        const long long tw = clk();
        mbar_wait(&tfull[r], rphase);
        e_w += clk() - tw;
        tc_fence_after();
        const uint32_t tcol = lane_base + r * BW;
        const long long tl0 = clk();
        uint32_t a[GPT][3][8];
        if (has_tile) {
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) tmem_ld8(tcol + (uint32_t)(kw * 16 + g_lo * 8), a[0][kw]);
          tmem_ld_wait();
          const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // zero the drained block for its next plane
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) tmem_st8(tcol + (uint32_t)(kw * 16 + g_lo * 8), z);
        }
        const long long tl1 = clk();
        e_ld += tl1 - tl0;
        if (live && has_tile) {
          // rows m+1 (kw 1) and m+2 (kw 2): shuffles within the quarter; lanes 30-31 take the
          // next quarter's rows 0-1 through shared memory (branch-free: every lane reads the
          // broadcast words, a select keeps them on lanes 30 / 31 only)
          float4* xw = reinterpret_cast<float4*>(&xch[hh][n & 1][q][0][0]);
          if (lane == 0) {
#pragma unroll
            for (int gi = 0; gi < GPT; ++gi) {
              xw[0 * 2 + 0] = make_float4(__uint_as_float(a[gi][1][0]), __uint_as_float(a[gi][1][1]),
                                                   __uint_as_float(a[gi][1][2]), __uint_as_float(a[gi][1][3]));
              xw[0 * 2 + 1] = make_float4(__uint_as_float(a[gi][1][4]), __uint_as_float(a[gi][1][5]),
                                                   __uint_as_float(a[gi][1][6]), __uint_as_float(a[gi][1][7]));
            }
          }
          if (lane < 2) {
#pragma unroll
            for (int gi = 0; gi < GPT; ++gi) {
              xw[(1 + lane) * 2 + 0] = make_float4(__uint_as_float(a[gi][2][0]), __uint_as_float(a[gi][2][1]),
                                                            __uint_as_float(a[gi][2][2]), __uint_as_float(a[gi][2][3]));
              xw[(1 + lane) * 2 + 1] = make_float4(__uint_as_float(a[gi][2][4]), __uint_as_float(a[gi][2][5]),
                                                            __uint_as_float(a[gi][2][6]), __uint_as_float(a[gi][2][7]));
            }
          }
          asm volatile("bar.sync %0, 128;" ::"r"(2 + hh) : "memory");
          const float4* xn = reinterpret_cast<const float4*>(&xch[hh][n & 1][q < 3 ? q + 1 : q][0][0]);
          const bool l31 = lane == 31, l30 = lane == 30;
#pragma unroll
          for (int gi = 0; gi < GPT; ++gi) {
            const int g = g_lo + gi;
            float xs[3][8];
#pragma unroll
            for (int sl = 0; sl < 3; ++sl) {
              const float4 u0 = xn[sl * 2 + 0], u1 = xn[sl * 2 + 1];
              xs[sl][0] = u0.x, xs[sl][1] = u0.y, xs[sl][2] = u0.z, xs[sl][3] = u0.w;
              xs[sl][4] = u1.x, xs[sl][5] = u1.y, xs[sl][6] = u1.z, xs[sl][7] = u1.w;
            }
            float s1[8], s2[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              s1[e] = __shfl_down_sync(0xffffffffu, __uint_as_float(a[gi][1][e]), 1);
              s2[e] = __shfl_down_sync(0xffffffffu, __uint_as_float(a[gi][2][e]), 2);
            }
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float t1 = l31 ? xs[0][e] : s1[e];
              const float t2 = l31 ? xs[2][e] : (l30 ? xs[1][e] : s2[e]);
              v[e] = __uint_as_float(a[gi][0][e]) + t1 + t2 + sbias[g * 8 + e];
            }
            if (p.flags & VM_CONV_MASK) {
              const uint32_t* mwv = reinterpret_cast<const uint32_t*>(&mk[gi]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                v[2 * e] = (int16_t)(mwv[e] & 0xFFFFu) > 0 ? v[2 * e] : 0.f;
                v[2 * e + 1] = (int16_t)(mwv[e] >> 16) > 0 ? v[2 * e + 1] : 0.f;
              }
            }
            int4 out;
            uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
            if (p.flags & VM_CONV_RELU) {
#pragma unroll
              for (int e = 0; e < 4; ++e) ow[e] = pack_bf16x2_relu(v[2 * e], v[2 * e + 1]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) ow[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
            }
            if (valid && g * 8 < p.Cout) {
              const int64_t orow = orow0 + (int64_t)o * p.P;
              *reinterpret_cast<int4*>(yb + g * p.plane8 + orow * 8) = out;
              if (HL && p.hl.lo && o == 0)
                *reinterpret_cast<int4*>(p.hl.lo + (yb - p.y) + g * p.plane8 + (orow + (int64_t)p.D * p.P) * 8) = out;
              if (HL && p.hl.hi && o == p.D - 1)
                *reinterpret_cast<int4*>(p.hl.hi + (yb - p.y) + g * p.plane8 + (orow - (int64_t)p.D * p.P) * 8) = out;
            }
          }
        }
        const long long tm1 = clk();
        tmem_st_wait();
        e_sw += clk() - tm1;
        if (DBG) e_m += tm1 - tl1;
        tc_fence_before();
        mbar_arrive(&tempty[r]);
        if (++r == (uint32_t)p.ring) {
          r = 0;
          rphase ^= 1u;
        }
      }
    }
    if (DBG && threadIdx.x == 96) {
      p.dbg[blockIdx.x * 8 + 4] = clk() - e0;
      p.dbg[blockIdx.x * 8 + 5] = e_w;
      p.dbg[blockIdx.x * 8 + 6] = (long long)n;
      p.dbg[blockIdx.x * 8 + 7] = e_ld * 1000000LL * 0 + e_ld;
    }
    if (DBG && threadIdx.x == 97) {  // sub-phases (kw_probe): exchange, math+store(+ld), st wait
      p.dbg[blockIdx.x * 8 + 1] = e_x;
      p.dbg[blockIdx.x * 8 + 2] = e_m;
      p.dbg[blockIdx.x * 8 + 3] = e_sw;
    }
  }
  tc_fence_before();
  if (HL && p.hl.counter) __threadfence();
  __syncthreads();
  if (HL && threadIdx.x == 0) halo_link_signal(p.hl);
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ weight gradient, kd along N
// Thin outputs (3*Nc <= 144): dW[kd,kh,kw][ci][co] = sum_a x[a + kd*P + kh*Wp + kw][ci] *
// gy[a + P + Wp + 1][co] is computed with kd moved to the B side: B = three gy slices shifted
// by -kd*P rows (N = 3*Nc, group (kd, cgo), one 16-byte-box TMA per kd with zero fill outside
// the sample), A = the runs-mode x staging without kd (M slot g = cg*3 + kh, kw = +16 B start).
// Per K step: 3 MMAs (one per kw, independent accumulators) of N = 3*Nc per M-tile, against
// 3 x 3 of N = Nc before.  The anchor range is extended to all Dp*P rows so every kd sees its
// full sum; anchors whose gy row falls in a margin or outside the sample contribute zero.
// A ones slot (g = 3*CG) yields the bias gradient in the kd = 0, kw = 0 block.
struct WkParams {
  const bf16* x;
  int64_t x_bstride;
  int64_t plane8;
  int B, P, Wp, rows;  // rows = Dp*P per sample
  int CG, CGo, Cout, Nc;
  int KS;              // anchors per stage (<= Wp - 2, multiple of 16)
  int MT, mt_per_unit, n_mtgroups;
  int nkw;             // kw taps per CTA (3, or 1 when 3 accumulators of N = 3*Nc exceed TMEM)
  int ngroups;         // CTA groups = n_mtgroups * (3 / nkw): (M-tile group, kw group)
  int ones_slot;
  int spk, ksplit, stages_total, units, grid, stages;
  int kinter;        // 1: stages interleaved over the split CTAs (L2 reuse of the kd slices)
  uint32_t a_bytes;
  uint32_t g_bytes;  // per kd slice: Nc/8 group slots of KS rows (CGo of them loaded)
  uint32_t g_load;   // loaded bytes per kd slice: CGo * KS * 16
  int ksub;              // K chunks of KS anchors per pipeline stage
  uint32_t sub_bytes;    // bytes per K chunk (A runs + 3 gy slices)
  uint32_t stage_bytes, idesc, idesc64;  // M = 64 for M-tiles with <= 8 live slots
  float* ws;  // [kidx][MT][3 kw][3*Nc][128]
  long long* dbg;  // optional cycle probes [gridDim][8] (vm_debug_set_fwd_probe)
};

// NMT: M-tiles of this CTA.  NKK > 0: K steps per chunk (KS/16), KSUB chunks per stage and
// all three kw taps, known at compile time so the MMA issue is straight-line code (measured:
// the runtime-bounded issue loop ran at ~39 cycles per M = 64, N = 48 MMA against 28);
// NKK = 0: runtime bounds.  Cycle probes when p.dbg is set.
template <int NMT, int NKK, int KSUB>
__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad_kd(const __grid_constant__ CUtensorMap gmap, const WkParams p) {
  const bool DBG = p.dbg != nullptr;
  auto clk = [DBG]() -> long long { return DBG ? (long long)clock64() : 0LL; };
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int grp = blockIdx.x % p.ngroups;      // (M-tile group, kw group) of this CTA
  const int mg_cta = grp % p.n_mtgroups;
  const int kw0 = (grp / p.n_mtgroups) * p.nkw;  // first kw tap of this CTA
  const int mt0 = mg_cta * p.mt_per_unit;
  const int nmt = min(p.mt_per_unit, p.MT - mt0);
  const int N3 = 3 * p.Nc;
  // slot i of this CTA's M-tiles sits at (i + slot_shift) * GS: runs of 3 slots (kh) per cg
  const int r0 = (16 * mt0) / 3;
  const int slot_shift = 16 * mt0 - 3 * r0;
  const uint32_t GS = (uint32_t)p.Wp * 16;
  // the CTA's last M-tile runs as M = 64 when it holds <= 8 live slots (ones slot included):
  // half the A-operand reads (TMEM rows m -> lanes (m/16)*32 + m%16)
  const bool last64 = 3 * p.CG + 1 - 16 * (mt0 + nmt - 1) <= 8;
  if (p.ones_slot >= 0 && p.ones_slot / 16 >= mt0 && p.ones_slot / 16 < mt0 + nmt) {
    const int local = p.ones_slot - mt0 * 16 + slot_shift;
    for (int s = 0; s < p.stages * p.ksub; ++s) {  // every K chunk of every stage
      uint32_t* dst = reinterpret_cast<uint32_t*>(smem + (size_t)(s / p.ksub) * p.stage_bytes +
                                                  (size_t)(s % p.ksub) * p.sub_bytes + (size_t)local * GS);
      for (int i = threadIdx.x; i < (p.KS + 8) * 4; i += blockDim.x) dst[i] = 0x3F803F80u;  // bf16 1.0 x2
    }
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  pdl_wait();  // dependents launch as this grid's CTAs exit (no early trigger)

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&gmap);
      int stage = 0;
      uint32_t phase = 0;
      const int r_end = min(p.CG - 1, (16 * (mt0 + nmt) - 1) / 3);  // last run of this CTA
      const int nrun = r_end >= r0 ? r_end - r0 + 1 : 0;
      const int Rrun = p.KS + 2 * p.Wp + 2;
      const uint32_t tx = p.ksub * ((uint32_t)nrun * Rrun * 16 + 3 * p.g_load);
      long long t_pe = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int ks = (u / p.ngroups) % p.ksplit;
        const int b = u / (p.ngroups * p.ksplit);
        // K stages interleaved over the split CTAs (stage s -> CTA s % ksplit): at any time the
        // CTAs read one contiguous window of rows, and the kd-shifted gy slices (1-2 planes back)
        // were read a few windows earlier by other CTAs: L2 hits instead of DRAM re-reads
        const int s0 = p.kinter ? ks : ks * p.spk, s1 = p.kinter ? p.stages_total : min(p.stages_total, s0 + p.spk);
        const int sstep = p.kinter ? p.ksplit : 1;
        const bf16* xb = p.x + b * p.x_bstride;
        for (int s = s0; s < s1; s += sstep) {
          const long long tw = clk();
          mbar_wait(&empty[stage], phase ^ 1);
          t_pe += clk() - tw;
          mbar_arrive_expect_tx(&full[stage], tx);
          for (int j = 0; j < p.ksub; ++j) {  // ksub consecutive K chunks per stage
            const int k0 = (s * p.ksub + j) * p.KS;
            uint8_t* sA = smem + (size_t)stage * p.stage_bytes + (size_t)j * p.sub_bytes;
            uint8_t* sG = sA + p.a_bytes;
            const int gr0 = k0 + p.P + p.Wp + 1;
            for (int kd = 0; kd < 3; ++kd)  // gy interior planes; other rows read as zeros
              tma_load_4d(sG + (size_t)kd * p.g_bytes, &gmap, &full[stage], 0, gr0 - (kd + 1) * p.P, 0, b);
            for (int r = r0; r <= r_end; ++r)
              bulk_load(sA + (size_t)(r - r0) * 3 * GS, xb + r * p.plane8 + (int64_t)k0 * 8, (uint32_t)Rrun * 16,
                        &full[stage]);
          }
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (p.dbg) p.dbg[blockIdx.x * 8 + 7] = t_pe;
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    bool started = false;
    const uint32_t id_last = last64 ? p.idesc64 : p.idesc;
    const long long t0 = clk();
    long long t_fu = 0, t_is = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int ks = (u / p.ngroups) % p.ksplit;
      // K stages interleaved over the split CTAs (stage s -> CTA s % ksplit): at any time the
      // CTAs read one contiguous window of rows, and the kd-shifted gy slices (1-2 planes back)
      // were read a few windows earlier by other CTAs: L2 hits instead of DRAM re-reads
      const int s0 = p.kinter ? ks : ks * p.spk, s1 = p.kinter ? p.stages_total : min(p.stages_total, s0 + p.spk);
      const int sstep = p.kinter ? p.ksplit : 1;
      for (int s = s0; s < s1; s += sstep) {
        const long long tf = clk();
        mbar_wait(&full[stage], phase);
        const long long tf1 = clk();
        t_fu += tf1 - tf;
        tc_fence_after();
        if (elect_one()) {
          const int ksub = NKK > 0 ? KSUB : p.ksub;
          const int nkk = NKK > 0 ? NKK : p.KS / 16;
          const int nkw = NKK > 0 ? 3 : p.nkw;
          const uint32_t sA0 = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t mstep = 16 * (GS >> 4);
#pragma unroll
          for (int j = 0; j < ksub; ++j) {
            const uint32_t sA = sA0 + (uint32_t)j * p.sub_bytes;
            const uint32_t sG = sA + p.a_bytes;
            // B: MN-major, N groups (kd, cgo) KS rows apart; A: MN-major slots GS apart
            const uint64_t b0desc = make_sdesc(sG, 128, (uint32_t)p.KS * 16);
            const uint64_t a0desc = make_sdesc(sA + (uint32_t)slot_shift * GS, 128, GS) + (uint64_t)kw0;
            const uint32_t acc0 = (started || j > 0) ? 1u : 0u;
#pragma unroll
            for (int kk = 0; kk < nkk; ++kk) {
              const uint64_t bdesc = b0desc + (uint64_t)(kk * 16);
              const uint32_t acc = kk > 0 ? 1u : acc0;
#pragma unroll
              for (int m = 0; m < NMT; ++m) {
                const uint64_t adesc = a0desc + (uint64_t)(m * mstep + kk * 16);
                const uint32_t d = tbase + (uint32_t)(m * nkw * N3);
                const uint32_t id = m == NMT - 1 ? id_last : p.idesc;
                mma_bf16_ss(d, adesc, bdesc, id, acc);
                if (nkw == 3) {
                  mma_bf16_ss(d + N3, adesc + 1, bdesc, id, acc);
                  mma_bf16_ss(d + 2 * N3, adesc + 2, bdesc, id, acc);
                }
              }
            }
          }
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        t_is += clk() - tf1;
        started = true;
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (elect_one()) mma_commit(&tfull);
    __syncwarp();
    if (p.dbg && lane == 0) {
      p.dbg[blockIdx.x * 8 + 0] = clk() - t0;
      p.dbg[blockIdx.x * 8 + 2] = t_fu;
      p.dbg[blockIdx.x * 8 + 3] = t_is;
    }
  } else {
    // drain: warp (2..5) reads TMEM lane quarter warp & 3
    const int q = warp & 3;
    const int kidx = blockIdx.x / p.ngroups;
    mbar_wait(&tfull, 0);
    tc_fence_after();
    for (int m = 0; m < nmt; ++m) {
      const bool m64 = last64 && m == nmt - 1;
      const int m_row = m64 ? q * 16 + lane : q * 32 + lane;
      const bool live = !m64 || lane < 16;
      for (int c0 = 0; c0 < p.nkw * N3; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(m * p.nkw * N3 + c0), r);
        tmem_ld_wait();
        float* dst = p.ws + (((int64_t)kidx * p.MT + mt0 + m) * 3 * N3 + kw0 * N3 + c0) * 128 + m_row;
        if (live) {
#pragma unroll
          for (int e = 0; e < 16; ++e) dst[e * 128] = __uint_as_float(r[e]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

}  // namespace vm

using namespace vm;

extern "C" size_t vm_packed_weights_bytes(int Cin, int Cout) {
  PackGeom g = pack_geom(Cin, Cout);
  return (size_t)g.nchunk * g.KC * 27 * 2 * g.Nc * 8 * sizeof(bf16);
}

// Batched repack of every layer's operands in one launch (after each SGD step): one thread
// per 16-byte output vector (8 input channels of one (tap, output channel)) over the
// concatenation of all jobs, the job found by binary search over the job offsets — load
// balanced across layers of very different sizes (a grid.y-per-job launch sized for the
// average job left the deep layers' blocks looping long after the thin ones were done).
// The decode runs once per vector and the fp32 reads are coalesced (plain: consecutive
// threads read consecutive co; flip: each thread reads 8 consecutive floats).
constexpr int kPackSmemJobs = 256;
__global__ void k_pack_batch(const vm_pack_job* __restrict__ jobs, int njobs, int64_t total) {
  // job offsets and layouts cached in shared memory (searched and decoded per vector)
  __shared__ int64_t sbegin[kPackSmemJobs];
  __shared__ PackGeom sgeom[kPackSmemJobs];
  const bool cached = njobs <= kPackSmemJobs;
  pdl_wait();
  if (cached) {
    for (int i = threadIdx.x; i < njobs; i += blockDim.x) {
      sbegin[i] = jobs[i].begin;
      sgeom[i] = jobs[i].flip ? pack_geom(jobs[i].cout, jobs[i].cin) : pack_geom(jobs[i].cin, jobs[i].cout);
    }
    __syncthreads();
  }
  for (int64_t gv = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gv < total / 8;
       gv += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = njobs - 1;  // last job with begin <= 8*gv
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((cached ? sbegin[mid] : jobs[mid].begin) <= gv * 8) lo = mid; else hi = mid - 1;
    }
    const vm_pack_job& jb = jobs[lo];
    const PackGeom g = cached ? sgeom[lo] : (jb.flip ? pack_geom(jb.cout, jb.cin) : pack_geom(jb.cin, jb.cout));
    const float* __restrict__ w = jb.w;
    const int64_t v = gv - jb.begin / 8;
    uint32_t r = (uint32_t)v;  // < 2^31 vectors per job (VM_REQUIRE at launch)
    int kd, kh, kw, kc, co, half;
    if (g.sweep == 2) {  // [kc][3 kh][2][144][8]
      const int n = (int)(r % 144u);
      r /= 144u;
      half = r & 1;
      r >>= 1;
      kh = (int)(r % 3u);
      kc = (int)(r / 3u);
      kd = 2 - n / 48;
      kw = (n % 48) / 16;
      co = n % 16;
    } else if (g.sweep) {
      const uint32_t N3 = 3u * g.Nc;
      const int n = (int)(r % N3);
      r /= N3;
      half = r & 1;
      r >>= 1;
      const int j = (int)(r % 9u);
      kc = (int)(r / 9u);
      kh = j / 3;
      kw = j % 3;
      kd = 2 - n / g.Nc;
      co = n % g.Nc;
    } else {
      const int n = (int)(r % (uint32_t)g.Nc);
      r /= (uint32_t)g.Nc;
      half = r & 1;
      r >>= 1;
      const int j = (int)(r % 9u);
      r /= 9u;
      kd = (int)(r % 3u);
      r /= 3u;
      kc = (int)(r % (uint32_t)g.KC);
      co = (int)(r / (uint32_t)g.KC) * g.Nc + n;
      kh = j / 3;
      kw = j % 3;
    }
    const int t = (kd * 3 + kh) * 3 + kw;
    const int ci0 = (kc * 2 + half) * 8;
    float f[8];
    if (!jb.flip) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        f[e] = (ci0 + e < g.cin && co < g.cout) ? w[((int64_t)t * jb.cin + ci0 + e) * jb.cout + co] : 0.f;
    } else {  // W'[t][ci'][co'] = W[26 - t][co'][ci']: 8 consecutive floats of row co'
      const float* src = w + ((int64_t)(26 - t) * jb.cin + co) * jb.cout + ci0;
      if (co < g.cout && ci0 + 8 <= g.cin && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        // two 16-byte loads instead of eight scalar ones (each lane reads its own row: the
        // scalar form made the kernel L1-wavefront bound)
        const float4 a = __ldg(reinterpret_cast<const float4*>(src));
        const float4 c = __ldg(reinterpret_cast<const float4*>(src + 4));
        f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = c.x, f[5] = c.y, f[6] = c.z, f[7] = c.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = (ci0 + e < g.cin && co < g.cout) ? src[e] : 0.f;
      }
    }
    uint4 o;
    o.x = pack_bf16x2(f[0], f[1]);
    o.y = pack_bf16x2(f[2], f[3]);
    o.z = pack_bf16x2(f[4], f[5]);
    o.w = pack_bf16x2(f[6], f[7]);
    reinterpret_cast<uint4*>(jb.packed)[v] = o;
  }
}

extern "C" int vm_pack_weights_batch(const vm_pack_job* jobs, int njobs, int64_t total_elems, void* stream) {
  VM_REQUIRE(jobs && njobs > 0 && total_elems > 0, VM_E_ARG, "vm_pack_weights_batch: bad argument");
  VM_REQUIRE(njobs <= 65535, VM_E_ARG, "vm_pack_weights_batch: too many jobs");
  VM_REQUIRE(total_elems / 8 < (1LL << 31), VM_E_SHAPE, "vm_pack_weights_batch: too many elements");
  launch_pdl(k_pack_batch, grid_for(total_elems / 8, 256), 256, 0, as_stream(stream), jobs, njobs, total_elems);
  return launch_status("vm_pack_weights_batch");
}

extern "C" int vm_pack_weights(const float* w, void* packed, int Cin, int Cout, int flip, void* stream) {
  VM_REQUIRE(w && packed && Cin > 0 && Cout > 0, VM_E_ARG, "vm_pack_weights: bad argument");
  PackGeom g = flip ? pack_geom(Cout, Cin) : pack_geom(Cin, Cout);
  int64_t total = (int64_t)vm_packed_weights_bytes(g.cin, g.cout) / 2;
  k_pack_weights<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(w, (bf16*)packed, g, Cin, Cout, flip);
  return launch_status("vm_pack_weights");
}

static long long* g_fwd_dbg = nullptr;
// Per host thread: SMs the forward / dgrad conv may occupy (0: all).  The interior-plane conv
// that overlaps a halo leaves a few SMs to the exchange's pack / NCCL / unpack kernels, which
// cannot co-reside with a 1-CTA-per-SM tensor-core conv (shared memory + TMEM).
static thread_local int g_conv_sm_limit = 0;
extern "C" int vm_set_conv_sm_limit(int n) {
  const int prev = g_conv_sm_limit;
  g_conv_sm_limit = n < 0 ? 0 : n;
  return prev;
}
static int g_sweep_xmode = 0;
extern "C" void vm_debug_set_sweep_mode(int m) { g_sweep_xmode = m; }
static int g_sweep_force_mb = 0;  // A/B probes: restrict the sweep planner to one MB
static int g_sweep_force_s = 0;   // A/B probes: restrict the sweep planner to one segment length
extern "C" void vm_debug_set_sweep_s(int sv) { g_sweep_force_s = sv; }
static int g_fwd_force_mb = 0, g_fwd_force_acc = 0;  // A/B probes: restrict the general fwd planner
extern "C" void vm_debug_set_fwd_plan(int mb, int nacc) { g_fwd_force_mb = mb, g_fwd_force_acc = nacc; }
extern "C" void vm_debug_set_sweep_mb(int mb) { g_sweep_force_mb = mb; }

// Plan + launch of the kd-stacked sweep kernel (weights packed with PackGeom::sweep).
// Units = (sample, column of MB*128 in-plane anchors, segment of S output planes); MB and
// S minimise waves * (S + 2) * MB, the MMA work per SM in tile-planes.
static int launch_sweep(const FwdParams& f, int nsm, void* stream) {
  SwParams p{};
  p.x = f.x;
  p.x_bstride = f.x_bstride;
  p.wpk = f.wpk;
  p.bias = f.bias;
  p.y = f.y;
  p.y_bstride = f.y_bstride;
  p.mask = f.mask;
  p.m_bstride = f.m_bstride;
  p.D = f.D;
  p.H = f.H;
  p.W = f.W;
  p.Hp = f.Hp;
  p.Wp = f.Wp;
  p.P = f.P;
  p.plane8 = f.plane8;
  p.CG = f.CG;
  p.KC = f.KC;
  p.Cout = f.Cout;
  p.Nc = f.Nc;
  p.flags = f.flags;
  p.dbg = f.dbg;
  p.hl = f.hl;
  p.xmode = g_sweep_xmode;
  p.w_bytes = (uint32_t)p.KC * 9 * 2 * 3 * p.Nc * 16;
  const int static_smem = 2 * 1024;
  // measured SS-mode tcgen05.mma cycles (tools/probes/probe_tput5, profiles/r01): one chain of
  // dependent accumulations costs ~68 cycles per MMA; >= 3 independent chains reach the
  // operand-bandwidth bound max(N/2, 32 + N/4)
  auto mma_cycles = [](int N, int chains) -> double {
    const double bw = N / 2.0 > 32 + N / 4.0 ? N / 2.0 : 32 + N / 4.0;
    if (chains >= 3) return bw + 1;
    if (chains == 2) return bw * 1.3 > 49 ? bw * 1.3 : 49;
    return bw > 68 ? bw : 68;
  };
  double best = 1e30;
  const bool kw = p.Nc == 16 && p.KC >= 2 && kSweepKw;  // packed as PackGeom::sweep == 2
  if (kw) {
    // N = 144 per MMA (3 kh x KC per plane and tile); tiles of 126 outputs; MB <= 2 (TMEM:
    // MB x ring x 48 columns, ring >= 4); 2 tiles = 2 independent accumulation chains
    for (int MB = 2; MB >= 1; --MB) {
      if (g_sweep_force_mb && MB != g_sweep_force_mb) continue;
      int ring = 512 / (MB * 48);
      if (ring > kSwMaxRing) ring = kSwMaxRing;
      const int R = MB * kKwTile + 2 + 2 * p.Wp;
      const uint32_t a_bytes = ((uint32_t)R * 16 + 127) & ~127u;
      const uint32_t stage_bytes = 2 * a_bytes;
      int stages = (int)((kSmemBudget - static_smem - (int)p.w_bytes) / (int)stage_bytes);
      if (stages > kSwMaxStages) stages = kSwMaxStages;
      if (stages < 3) continue;
      const int ncol = (p.P + MB * kKwTile - 1) / (MB * kKwTile);
      // two of every `ring` planes split at the ring end (two MMAs per kh)
      const double wrapf = 1.0 + 2.0 * 0.39 / ring;
      const double plane = 3.0 * p.KC * MB * mma_cycles(144, MB >= 2 ? 3 : 1) * wrapf + 900.0;
      for (int S = 1; S <= p.D; ++S) {
        if (g_sweep_force_s && S != g_sweep_force_s && g_sweep_force_s <= p.D) continue;
        const int nseg = (p.D + S - 1) / S;
        const int64_t units = (int64_t)f.B * ncol * nseg;
        const int64_t waves = (units + nsm - 1) / nsm;
        const double cost = (double)waves * (S + 3) * plane;
        if (cost < best) {
          best = cost;
          p.MB = MB, p.ring = ring, p.R = R, p.a_bytes = a_bytes, p.stage_bytes = stage_bytes;
          p.stages = stages, p.ncol = ncol, p.S = S, p.nseg = nseg, p.units = (int)units;
        }
      }
    }
    VM_REQUIRE(best < 1e30, VM_E_UNSUPPORTED, "vm_conv3d_fwd_tc: no sweep-kw configuration fits (W=%d)", p.W);
    p.idesc1 = make_idesc_bf16(128, 48, false, false);
    p.idesc2 = make_idesc_bf16(128, 96, false, false);
    p.idesc3 = make_idesc_bf16(128, 144, false, false);
    const size_t smem = (size_t)p.w_bytes + (size_t)p.stages * p.stage_bytes;
    const int grid = p.units < nsm ? p.units : nsm;
    const int mode = p.dbg != nullptr ? 1 : (p.hl.counter || p.hl.wait_own) ? 2 : 0;
    using SwKern = void (*)(const SwParams);
    static const SwKern ktable[2][3] = {
        {k_conv_fwd_sweepkw<1, 0>, k_conv_fwd_sweepkw<1, 1>, k_conv_fwd_sweepkw<1, 2>},
        {k_conv_fwd_sweepkw<2, 0>, k_conv_fwd_sweepkw<2, 1>, k_conv_fwd_sweepkw<2, 2>}};
    auto kern = ktable[p.MB - 1][mode];
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, grid, kKwThreads, smem, as_stream(stream), p);
    return launch_status("vm_conv3d_fwd_tc (sweep-kw)");
  }
  for (int MB = 4; MB >= 1; --MB) {
    if (g_sweep_force_mb && MB != g_sweep_force_mb) continue;
    int ring = 512 / (MB * p.Nc);
    if (ring > kSwMaxRing) ring = kSwMaxRing;
    if (ring < 4) continue;
    const int R = MB * 128 + 2 * p.Wp + 2;
    const uint32_t a_bytes = ((uint32_t)R * 16 + 127) & ~127u;
    const uint32_t stage_bytes = 2 * a_bytes;
    int stages = (int)((kSmemBudget - static_smem - (int)p.w_bytes) / (int)stage_bytes);
    if (stages > kSwMaxStages) stages = kSwMaxStages;
    if (stages < 3) continue;
    const int ncol = (p.P + MB * 128 - 1) / (MB * 128);
    // per input plane: 9*KC MMAs per tile (+1 at the first K step); a short ring (< 6) stalls
    // + ~900 cycles of per-plane MMA-warp bookkeeping (measured with tools/dbg_sweep_probe.py)
    const double plane = (9.0 * p.KC + 1) * MB * mma_cycles(3 * p.Nc, MB) * (ring < 6 ? 1.15 : 1.0) + 900.0;
    for (int S = 1; S <= p.D; ++S) {
      if (g_sweep_force_s && S != g_sweep_force_s && g_sweep_force_s <= p.D) continue;
      const int nseg = (p.D + S - 1) / S;
      const int64_t units = (int64_t)f.B * ncol * nseg;
      const int64_t waves = (units + nsm - 1) / nsm;
      const double cost = (double)waves * (S + 3) * plane;  // + ~1 plane of pipeline fill
      if (cost < best) {
        best = cost;
        p.MB = MB;
        p.ring = ring;
        p.R = R;
        p.a_bytes = a_bytes;
        p.stage_bytes = stage_bytes;
        p.stages = stages;
        p.ncol = ncol;
        p.S = S;
        p.nseg = nseg;
        p.units = (int)units;
      }
    }
  }
  VM_REQUIRE(best < 1e30, VM_E_UNSUPPORTED, "vm_conv3d_fwd_tc: no sweep configuration fits (W=%d)", p.W);
  p.idesc1 = make_idesc_bf16(128, p.Nc, false, false);
  p.idesc2 = make_idesc_bf16(128, 2 * p.Nc, false, false);
  p.idesc3 = make_idesc_bf16(128, 3 * p.Nc, false, false);
  const size_t smem = (size_t)p.w_bytes + (size_t)p.stages * p.stage_bytes;
  const int grid = p.units < nsm ? p.units : nsm;
  const bool dbg = p.dbg != nullptr;
  using SwKern = void (*)(const SwParams);
#define SW_ROW(MB_)                                                                                   \
  {k_conv_fwd_sweep<MB_, 0, 2>, k_conv_fwd_sweep<MB_, 0, 4>, k_conv_fwd_sweep<MB_, 0, 6>, \
   k_conv_fwd_sweep<MB_, 1, 2>, k_conv_fwd_sweep<MB_, 1, 4>, k_conv_fwd_sweep<MB_, 1, 6>, \
   k_conv_fwd_sweep<MB_, 2, 2>, k_conv_fwd_sweep<MB_, 2, 4>, k_conv_fwd_sweep<MB_, 2, 6>}
  static const SwKern table[4][9] = {SW_ROW(1), SW_ROW(2), SW_ROW(3), SW_ROW(4)};
#undef SW_ROW
  VM_REQUIRE(p.Nc == 16 || p.Nc == 32 || p.Nc == 48, VM_E_UNSUPPORTED, "sweep conv: Nc %d", p.Nc);
  const bool hl = p.hl.counter || p.hl.wait_own;
  auto kern = table[p.MB - 1][(dbg ? 3 : hl ? 6 : 0) + p.Nc / 16 - 1];
  const cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = (p.MB == 4 && p.Nc == 16) ? sweep_threads<4, 2>() : sweep_threads<1, 4>() + (p.MB >= 2 ? 32 : 0);
  VM_REQUIRE(ea == cudaSuccess, 100 + (int)ea, "sweep: smem attribute %zu B (MB %d, S %d, ring %d, stages %d): %s",
             smem, p.MB, p.S, p.ring, p.stages, cudaGetErrorString(ea));
  launch_pdl(kern, grid, threads, smem, as_stream(stream), p);
  {
    const cudaError_t el = cudaPeekAtLastError();
    VM_REQUIRE(el == cudaSuccess, 100 + (int)el, "sweep launch: grid %d x %d threads, smem %zu (MB %d S %d ring %d stages %d units %d): %s",
               grid, threads, smem, p.MB, p.S, p.ring, p.stages, p.units, cudaGetErrorString(el));
  }
  return launch_status("vm_conv3d_fwd_tc (sweep)");
}

extern "C" void vm_debug_set_fwd_probe(long long* buf) { g_fwd_dbg = buf; }

static void (*fwd_kernel(int MB, int mode))(const FwdParams) {
#define FWD_ROW(M) {k_conv_fwd_tc<M, 0>, k_conv_fwd_tc<M, 1>, k_conv_fwd_tc<M, 2>}
  static void (*const ftable[8][3])(const FwdParams) = {FWD_ROW(1), FWD_ROW(2), FWD_ROW(3), FWD_ROW(4),
                                                        FWD_ROW(5), FWD_ROW(6), FWD_ROW(7), FWD_ROW(8)};
#undef FWD_ROW
  return ftable[(MB < 1 ? 1 : MB > 8 ? 8 : MB) - 1][mode];
}

// Split-K workspace of the general forward kernel: [tile-unit counters (256 B aligned)]
// [f32 partials ksplit x tile units x MB x Nc x 128].  Zeroed once by the caller.
static size_t fwd_ws_need(int ksplit, int64_t ntu, int MB, int Nc) {
  if (ksplit <= 1) return 0;
  return (size_t)((ntu * 8 + 255) / 256 * 256) + (size_t)ksplit * ntu * MB * Nc * 128 * sizeof(float);
}
// Split-K is off by default: measured on B200 it loses at every deep-level shape of the cfg2
// ladder (128->128 @16^3: 19.1 us unsplit, 24.9 / 26.6 us with 2 / 3 splits — the partial
// round trip and the last split's fix-up cost more than the shorter K loop saves).
// Split-K is planned only for layers with few tile units (<= SMs / 4): the deep levels of a
// split volume (cfg3 8-way, level 4: 2x16x16 local, 512 channels: 12 units of 96 K stages);
// at cfg2's deep levels (41 units) it lost (see below) and stays off by that rule
static int g_fwd_max_split = kFwdMaxSplit;  // vm_debug_set_fwd_max_split (A/B probes, tests)
extern "C" void vm_debug_set_fwd_max_split(int v) { g_fwd_max_split = v < 1 ? 1 : v > kFwdMaxSplit ? kFwdMaxSplit : v; }
static int g_fwd_force_split = 0;  // vm_debug_force_fwd_split (plan sweeps): only this K split
// Cluster split-K is opt-in (vm_debug_set_fwd_cluster(1)): alone it beats the global fix-up at
// 2-4 splits (128->128 @16^3 split 3: 15.2 vs 16.8 us; 256->256 @4x32^2 split 4: 28.7 vs 28.9),
// bitwise the same result, but inside the step it lost (cfg2 2.728 vs 2.70 ms): a cluster needs
// ksplit SMs of one GPC free at once while the weight-gradient stream's CTAs hold SMs.
static int g_fwd_cluster = 0;
extern "C" void vm_debug_set_fwd_cluster(int on) { g_fwd_cluster = on; }
static void (*fwd_kernel(int MB, int mode))(const FwdParams);
// clusters of `size` fwd CTAs (one per SM: TMEM + shared memory) that can be resident at once: a
// GPC holds whole clusters only, so 4-CTA clusters leave SMs idle and a plan with more units
// than this would run a second wave (768->256 @4x32^2, split 4: 85 vs 48 us)
static int fwd_max_clusters(int MB, int size, size_t smem) {
  static int cache[9][9] = {};
  if (size < 2 || size > 8 || MB < 1 || MB > 8) return 0;
  int& c = cache[MB][size];
  if (c == 0) {
    auto kern = fwd_kernel(MB, 0);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(size * 16);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = kSmemBudget;  // every plan's stages fill the budget: 1 CTA per SM
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = -1;  // unknown: no cluster plans
    }
    c = n;
  }
  (void)smem;
  return c;
}
extern "C" void vm_debug_force_fwd_split(int v) { g_fwd_force_split = v; }

static int fwd_tc_launch(const void* x, int64_t x_bstride, const void* wpacked, const float* bias, void* y,
                         int64_t y_bstride, const void* mask, int64_t mask_bstride, int B, int Cin, int Cout, int D,
                         int H, int W, unsigned flags, void* ws, size_t ws_bytes, void* stream, int Dfull = 0,
                         const vm_halo_link* link = nullptr);

extern "C" int vm_conv3d_fwd_tc(const void* x, int64_t x_bstride, const void* wpacked,
                                const float* bias, void* y, int64_t y_bstride, const void* mask,
                                int64_t mask_bstride, int B, int Cin, int Cout, int D, int H, int W,
                                unsigned flags, void* stream) {
  return fwd_tc_launch(x, x_bstride, wpacked, bias, y, y_bstride, mask, mask_bstride, B, Cin, Cout, D, H, W, flags,
                       nullptr, 0, stream);
}

extern "C" int vm_conv3d_fwd_tc_ws(const void* x, int64_t x_bstride, const void* wpacked, const float* bias,
                                   void* y, int64_t y_bstride, const void* mask, int64_t mask_bstride, int B,
                                   int Cin, int Cout, int D, int H, int W, unsigned flags, void* ws,
                                   size_t ws_bytes, void* stream) {
  return fwd_tc_launch(x, x_bstride, wpacked, bias, y, y_bstride, mask, mask_bstride, B, Cin, Cout, D, H, W, flags,
                       ws, ws_bytes, stream);
}

extern "C" int vm_conv3d_fwd_tc_link(const void* x, int64_t x_bstride, const void* wpacked, const float* bias,
                                     void* y, int64_t y_bstride, const void* mask, int64_t mask_bstride, int B,
                                     int Cin, int Cout, int D, int H, int W, unsigned flags, void* ws,
                                     size_t ws_bytes, const vm_halo_link* link, void* stream) {
  return fwd_tc_launch(x, x_bstride, wpacked, bias, y, y_bstride, mask, mask_bstride, B, Cin, Cout, D, H, W, flags,
                       ws, ws_bytes, stream, 0, link);
}

// Output planes [d0, d0 + nd) of a slab with D interior planes: the conv of a plane reads
// input planes d-1..d+1 only, so the interior planes [1, D-1) can run while a halo exchange
// fills the margin planes, and the two boundary planes after it (north-star
// subsystem 2: exchange overlapped with interior-tile compute).
extern "C" int vm_conv3d_fwd_tc_range(const void* x, int64_t x_bstride, const void* wpacked, const float* bias,
                                      void* y, int64_t y_bstride, const void* mask, int64_t mask_bstride, int B,
                                      int Cin, int Cout, int D, int H, int W, int d0, int nd, unsigned flags,
                                      void* ws, size_t ws_bytes, void* stream) {
  VM_REQUIRE(d0 >= 0 && nd > 0 && d0 + nd <= D, VM_E_SHAPE, "vm_conv3d_fwd_tc_range: planes [%d,%d) outside [0,%d)",
             d0, d0 + nd, D);
  const int64_t off = (int64_t)d0 * (H + 2) * (W + 2) * 8;
  const bf16* xb = static_cast<const bf16*>(x) + off;
  bf16* yb = static_cast<bf16*>(y) + off;
  const bf16* mb = mask ? static_cast<const bf16*>(mask) + off : nullptr;
  if (!x_bstride) x_bstride = default_bstride(Cin, D, H, W, 1);
  if (!y_bstride) y_bstride = default_bstride(Cout, D, H, W, 1);
  if (mask && !mask_bstride) mask_bstride = default_bstride(Cout, D, H, W, 1);
  return fwd_tc_launch(xb, x_bstride, wpacked, bias, yb, y_bstride, mb, mask_bstride, B, Cin, Cout, nd, H, W, flags,
                       ws, ws_bytes, stream, D);
}

// Upper bound of the split-K workspace any plan of this shape may use (0: never splits).
extern "C" size_t vm_conv3d_fwd_tc_ws_bytes(int B, int Cin, int Cout, int D, int H, int W) {
  const PackGeom pg = pack_geom(Cin, Cout);
  if (pg.sweep) return 0;
  const int64_t tiles = ((int64_t)D * (H + 2) * (W + 2) + 127) / 128;
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  if ((int64_t)B * tiles * pg.nchunk * 4 > nsm * 8) return 256;  // never split (planner rule, MB <= 8)
  // MB tiles per unit round the tile count up by < MB tiles: bound by MB = 1 plus 8 tiles
  return fwd_ws_need(kFwdMaxSplit, (int64_t)B * (tiles + 8) * pg.nchunk, 1, pg.Nc) + 256;
}

// Dfull > 0: the slabs hold Dfull interior planes and D is a sub-range of output planes whose
// first plane the caller has already offset x / y / mask to (vm_conv3d_fwd_tc_range): the
// channel-group plane stride and the default batch strides come from Dfull.
static int fwd_tc_launch(const void* x, int64_t x_bstride, const void* wpacked, const float* bias, void* y,
                         int64_t y_bstride, const void* mask, int64_t mask_bstride, int B, int Cin, int Cout, int D,
                         int H, int W, unsigned flags, void* ws, size_t ws_bytes, void* stream, int Dfull,
                         const vm_halo_link* link) {
  if (Dfull <= 0) Dfull = D;
  VM_REQUIRE(!link || Dfull == D, VM_E_ARG, "vm_conv3d_fwd_tc_link: a halo link needs the full plane range");
  VM_REQUIRE(!link || ((!link->push_lo && !link->push_hi) || (link->counter && link->epoch)) &&
                          (!link->wait_own || link->epoch),
             VM_E_ARG, "vm_conv3d_fwd_tc_link: incomplete halo link");
  VM_REQUIRE(x && wpacked && y, VM_E_ARG, "vm_conv3d_fwd_tc: null pointer");
  VM_REQUIRE((flags & VM_CONV_NOBIAS) || bias, VM_E_ARG, "vm_conv3d_fwd_tc: bias required");
  VM_REQUIRE(!(flags & VM_CONV_MASK) || mask, VM_E_ARG, "vm_conv3d_fwd_tc: mask required");
  VM_REQUIRE(B > 0 && Cin > 0 && Cout > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE,
             "vm_conv3d_fwd_tc: bad shape");
  PackGeom pg = pack_geom(Cin, Cout);
  FwdParams p{};
  p.hl = halo_link_of(link);
  p.wpk = static_cast<const bf16*>(wpacked);
  p.bias = bias;
  p.y = static_cast<bf16*>(y);
  p.mask = static_cast<const bf16*>(mask);
  p.B = B;
  p.D = D;
  p.H = H;
  p.W = W;
  p.Hp = H + 2;
  p.Wp = W + 2;
  p.P = p.Hp * p.Wp;
  p.anchors = (int64_t)D * p.P;
  const int64_t rows = (int64_t)(Dfull + 2) * p.P;
  p.plane8 = rows * 8;
  p.y_bstride = y_bstride ? y_bstride : default_bstride(Cout, Dfull, H, W, 1);
  p.m_bstride = mask_bstride ? mask_bstride : default_bstride(Cout, Dfull, H, W, 1);
  p.CG = pg.CG;
  p.KC = pg.KC;
  p.Cout = Cout;
  p.Nc = pg.Nc;
  p.nchunk = pg.nchunk;
  p.flags = flags | (pdl_late() ? kFlagPdlLate : 0u);
  p.dbg = g_fwd_dbg;
  p.wp_magic = (uint32_t)(0x100000000ULL / (uint64_t)(W + 2)) + 1;
  p.hp_magic = (uint32_t)(0x100000000ULL / (uint64_t)(H + 2)) + 1;
  p.x = static_cast<const bf16*>(x);
  p.x_bstride = x_bstride ? x_bstride : default_bstride(Cin, Dfull, H, W, 1);
  VM_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (p.x_bstride & 7) == 0, VM_E_ALIGN,
             "vm_conv3d_fwd_tc: slab must be 16-byte aligned");
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  if (g_conv_sm_limit > 0 && g_conv_sm_limit < nsm) nsm = g_conv_sm_limit;
  if (pg.sweep) return launch_sweep(p, nsm, stream);
  p.b_bytes = 9 * 2 * p.Nc * 16;
  const int N = p.Nc;  // accumulator columns per tile
  const int tiles = (int)((p.anchors + 127) / 128);
  // Plan (MB tiles per unit, nacc accumulator sets, nbuf TMEM buffers) by a cost model of the
  // measured B200 behaviour: an MMA waits for the previous one into the same accumulator
  // (~68+ cycles), >= 3 independent chains reach max(N/2, 32 + N/4) cycles (tools/probes,
  // profiles/r01/probe_tput5.txt); a stage also pays its shared-memory traffic (TMA writes +
  // operand reads at ~128 B/clk).  Units = tiles/MB spread over the SMs in waves.
  auto mma_cycles = [](int n, int chains) -> double {
    const double bw = n / 2.0 > 32 + n / 4.0 ? n / 2.0 : 32 + n / 4.0;
    // below N = 256 the stage's shared-memory traffic hides the accumulator dependency: forced
    // plans (tools/dbg_fwd_plan.py) ran nacc = 1 as fast as or faster than nacc = 3 at N = 32..128
    // (the extra sets only cost TMEM drain: 128->128 @16^3 15.9 vs 16.2 us, 96->32 @64^3 68.6 vs
    // 77.9 us); the chain model (probe_tput5, an MMA-only loop) applies at N = 256
    if (chains >= 3 || n < 256) return bw + 1;
    if (chains == 2) return bw * 1.3 > 49 ? bw * 1.3 : 49;
    return bw > 68 ? bw * 1.5 : 68;
  };
  double best = 1e30;
  int bMB = 1, bacc = 1, bbuf = 1, bstages = 0, bsplit = 1;
  bool bcluster = false;
  for (int MB = 1; MB <= 8; ++MB) {
    if (g_fwd_force_mb && MB != g_fwd_force_mb) continue;
    const int R = MB * 128 + 2 * p.Wp + 2;
    const uint32_t a_bytes = (uint32_t)((R + 7) / 8 * 8) * 16;
    const uint32_t stage_bytes = 2 * a_bytes + p.b_bytes;
    int stages = kSmemBudget / (int)stage_bytes;
    if (stages > kMaxStages) stages = kMaxStages;
    if (stages < 2) continue;
    const int64_t ntu = (int64_t)B * ((tiles + MB - 1) / MB) * p.nchunk;
    // split-K over the 3*KC (kc, kd) stages when a caller workspace can hold the f32
    // partials: more CTAs for layers with few tiles (deep levels)
    for (int ksplit = 1; ksplit <= g_fwd_max_split; ++ksplit) {
      if (g_fwd_force_split && ksplit != g_fwd_force_split) continue;
      // cluster split: the ksplit CTAs of a tile unit form one cluster (<= 8, portable size),
      // one unit per CTA, the f32 partial tile fits the CTA's stage buffers
      // (<= 4: at 6-8 splits the global fix-up measured faster, tools/split_check.py)
      const bool cl = g_fwd_cluster && ksplit > 1 && ksplit <= 4 && ntu * ksplit <= nsm &&
                      (int64_t)MB * 128 * N * 4 <= (int64_t)stages * stage_bytes &&
                      ntu <= fwd_max_clusters(MB, ksplit, (size_t)stages * stage_bytes);
      if (ksplit > 1 && ntu * 4 > nsm && !cl && !g_fwd_force_split) break;  // enough tile units already
      // split plans with MB > 1 lost to MB = 1 at every forced-plan shape (tools/fwd_plan_sweep.py:
      // 256->256 @8^3 split 12: 28.3 vs 19.4 us; 512->512 @2x16^2: 34.7 vs 24.5 us)
      if (ksplit > 1 && MB > 1 && !g_fwd_force_split) break;
      const int spk = (3 * p.KC + ksplit - 1) / ksplit;
      if (ksplit > 1 && ((3 * p.KC + spk - 1) / spk != ksplit ||
                         (!cl && (!ws || fwd_ws_need(ksplit, ntu, MB, N) > ws_bytes))))
        continue;
      const int64_t units = ntu * ksplit;
      // the splits of a tile finish it together (they wait for each other): one wave only
      if (ksplit > 1 && units > nsm) break;
      const int64_t waves = (units + nsm - 1) / nsm;
      for (int nacc : {1, 2, 3}) {
        if (g_fwd_force_acc && nacc != g_fwd_force_acc) continue;
        for (int nbuf = 2; nbuf >= 1; --nbuf) {
          if (nbuf * MB * nacc * N > 512) continue;
          const double mma = 9.0 * MB * mma_cycles(N, MB * nacc);
          const double smem = (2.0 * R * 16 + p.b_bytes + 9.0 * MB * (4096 + 32.0 * N)) / 128.0;
          const double stage = mma > smem ? mma : smem;
          // single-buffered TMEM: the epilogue drain is not overlapped (~600 cycles per
          // 8-channel group and thread, measured with tools/dbg_fwd_probe.py; 200 made the
          // planner pick MB = 5 single-buffered for 32->96 at 64^3: 64.9 us vs 48.4 at MB = 2)
          // TMEM reads at 64 B/clk per SM (B300_MICROARCH: LDTM throughput) bound the drain of
          // MB x nacc x N f32 columns of 128 lanes; the last unit's drain is never overlapped
          const double drain_one = std::max(MB * (N / 8.0) * 600.0 / (MB > 1 ? 2 : 1),
                                            MB * nacc * N * 128.0 * 4.0 / 64.0);
          const double drain = nbuf == 1 ? drain_one : drain_one / (double)waves;
          // split: partial write, the wait for the tile's other splits, then each split CTA
          // sums its 1/ksplit of the rows: 256 (row, group) items in flight, 4 splits' loads
          // per round trip (~800 cycles from L2)
          const double fix_items = MB * std::ceil(128.0 / ksplit) * (N / 8.0);
          // cluster: drain into shared memory, two cluster barriers, DSMEM reads.  The constant
          // terms are fitted to forced plans (tools/split_check.py: 128->128 and 64->128 at 16^3,
          // unsplit vs split 3 — ~11 K cycles of split overhead, cluster, ~14 K global)
          const double fix = ksplit <= 1 ? 0.0
                             : cl ? 8000.0 + MB * (N / 8.0) * 60.0 +
                                        std::ceil(fix_items / 256.0) * std::ceil(ksplit / 4.0) * 600.0
                                  : 10000.0 + MB * (N / 8.0) * 60.0 +
                                        std::ceil(fix_items / 256.0) * std::ceil(ksplit / 4.0) * 800.0;
          const double cost = (double)waves * ((double)spk * stage + drain + fix + 2000.0);
          if (cost < best * 0.999) {
            best = cost;
            bMB = MB, bacc = nacc, bbuf = nbuf, bstages = stages, bsplit = ksplit, bcluster = cl;
          }
        }
      }
    }
  }
  VM_REQUIRE(bstages >= 2, VM_E_UNSUPPORTED, "vm_conv3d_fwd_tc: W=%d too wide for the stage budget", W);
  p.MB = bMB;
  p.nacc = bacc;
  p.nbuf = bbuf;
  p.R = p.MB * 128 + 2 * p.Wp + 2;
  p.Ralloc = (p.R + 7) / 8 * 8;
  p.a_bytes = (uint32_t)p.Ralloc * 16;
  p.stage_bytes = 2 * p.a_bytes + p.b_bytes;
  p.stages = bstages;
  p.mblocks = (tiles + p.MB - 1) / p.MB;
  p.ksplit = bsplit;
  p.spk = (3 * p.KC + bsplit - 1) / bsplit;
  p.units = B * p.mblocks * p.nchunk * bsplit;
  p.cluster = bcluster ? 1 : 0;
  if (bsplit > 1 && !bcluster) {
    const int64_t ntu = (int64_t)B * p.mblocks * p.nchunk;
    p.counters = static_cast<int*>(ws);  // [ntu] arrivals, [ntu] departures
    p.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + (ntu * 8 + 255) / 256 * 256);
  }
  p.idesc = make_idesc_bf16(128, N, false, false);
  (void)rows;
  const size_t smem = (size_t)p.stages * p.stage_bytes;
  int grid = p.units < nsm ? p.units : nsm;
  void (*kern)(const FwdParams) = nullptr;
  const int mode = p.dbg != nullptr ? 1 : (p.hl.counter || p.hl.wait_own) ? 2 : 0;
  kern = fwd_kernel(p.MB, mode);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (p.cluster) {  // one unit per CTA, clusters of the ksplit CTAs of a tile unit
    VM_REQUIRE(p.units <= nsm && p.units % p.ksplit == 0, VM_E_UNSUPPORTED, "fwd cluster split: %d units", p.units);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.units);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)p.ksplit;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, p);
    return launch_status("vm_conv3d_fwd_tc (cluster split)");
  }
  launch_pdl(kern, grid, 320, smem, as_stream(stream), p);
  return launch_status("vm_conv3d_fwd_tc");
}


namespace {
struct WgPlan {
  WgParams p;
  size_t ws_main, ws_bias;
};

int g_force_runs = -1, g_force_ks = 0, g_force_mpu = 0;  // tools/tune_wgrad.py overrides
int g_wg_chunk = 1;  // vm_debug_set_wgrad_chunk (A/B of the input-channel chunks; 2: any volume)
int g_wg_merge = 1;  // vm_debug_set_wgrad_merge (A/B: output chunks as one launch vs one call each)
constexpr int kWgradMaxCout = 160, kWgradChunk = 128;
// Cout > 160 in whole 128-channel chunks: one launch, chunk = CTA column (else one call per chunk)
static bool wgrad_merged_chunks(int Cout) {
  return g_wg_merge && Cout > kWgradMaxCout && Cout % kWgradChunk == 0;
}
thread_local int g_wg_phase = 0;  // vm_conv3d_wgrad_tc_phase: 0 all, 1 main kernel(s), 2 finalize
// splits bias_grad_partial_bf16 uses for this shape (the finalize's phase needs the count only)
static int bias_grad_partial_count(int B, int Cout, int D, int H, int W) {
  return (int)(bias_grad_ws_bytes((int64_t)B * D * H * W, Cout) / (((Cout + 7) / 8) * 8 * sizeof(float)));
}
int g_wg_interleave = 1;  // vm_debug_set_wgrad_interleave: 0 never, 1 planner's choice, 2 always (A/B)
int g_wg_min_spk = 2;  // minimum stages per K-split unit (vm_debug_set_wgrad_min_spk)
int g_wk_runtime = 0;  // 1: force the runtime-bounded kd wgrad issue loop (A/B probe)
int g_wk_ksub_min_stages = 2;  // two K chunks per stage when this many stages still fit (measured: 2 best)

int plan_wgrad(int B, int Cin, int Cout, int D, int H, int W, WgPlan& pl) {
  WgParams& p = pl.p;
  p = WgParams{};
  p.B = B;
  p.D = D;
  p.H = H;
  p.W = W;
  p.Hp = H + 2;
  p.Wp = W + 2;
  p.P = p.Hp * p.Wp;
  const int64_t rows = (int64_t)(D + 2) * p.P;
  p.plane8 = rows * 8;
  p.CG = (Cin + 7) / 8;
  p.Cout = Cout;
  // wide layers: output chunks of 128 channels (3 kw x 128 TMEM columns per M-tile) as
  // independent CTA columns of ONE launch
  p.nchunk = wgrad_merged_chunks(Cout) ? Cout / kWgradChunk : 1;
  p.Nc = p.nchunk > 1 ? kWgradChunk : (Cout + 15) / 16 * 16;
  p.NcTot = p.nchunk * p.Nc;
  p.CGo = p.nchunk > 1 ? p.Nc / 8 : (Cout + 7) / 8;
  VM_REQUIRE(3 * p.Nc <= 512, VM_E_UNSUPPORTED, "vm_conv3d_wgrad_tc: Cout %d > 160 not supported yet", Cout);
  p.MT = (9 * p.CG + 15) / 16;
  p.ones_slot = (9 * p.CG) % 16 ? 9 * p.CG : -1;
  p.gwide = rows % 8 == 0 ? 1 : 0;
  p.gdelta = p.gwide ? (int)((p.P + p.Wp + 1) & 7) : 0;
  p.mt_per_unit = 512 / (3 * p.Nc);
  if (p.mt_per_unit > p.MT) p.mt_per_unit = p.MT;
  // Plan rule, tuned on B200 (tools/tune_wgrad.py): the TMA request count dominates, so
  //  * rows wide enough (KS = 16*floor((Wp-2)/16) >= 32): "runs" staging, as many M-tiles per
  //    unit as fit in a double-buffered stage;
  //  * otherwise one copy per slot with the longest K chunk that double-buffers at 1 M-tile.
  const int ks_opts[4] = {256, 192, 128, 64};
  const int mpu_max = p.mt_per_unit;
  const int ks_run = min(256, ((p.Wp - 2) / 16) * 16);
  int best_mpu = 0, best_ks = 0, best_runs = 0;
  auto g_region = [&](int KS) -> uint32_t {  // gy bytes per stage (Nc/8 group slots)
    return (uint32_t)(p.Nc / 8) * (KS + 8) * 16;
  };
  auto fits = [&](int runs, int KS, int mpu) {
    const int RR = KS + 8;
    if (!p.gwide && RR > 256) return false;
    const int ralloc = (16 * mpu + 2) / 3 + 2;
    const uint32_t a_b = ((runs ? (uint32_t)ralloc * 3 * p.Wp * 16 : (uint32_t)mpu * 16 * RR * 16) + 1023) & ~1023u;
    const uint32_t stage = (a_b + g_region(KS) + 1023) & ~1023u;
    return kSmemBudget / (int)stage >= 2;
  };
  auto forced_ok = [&](int runs, int KS, int mpu) {
    return !((g_force_runs >= 0 && g_force_runs <= 1 && runs != g_force_runs) || (g_force_ks && KS != g_force_ks) ||
             (g_force_mpu && mpu != g_force_mpu));
  };
  if (ks_run >= 64 && g_force_runs != 0) {
    for (int mpu = mpu_max; mpu >= 1 && !best_mpu; --mpu)
      if (fits(1, ks_run, mpu) && forced_ok(1, ks_run, mpu)) {
        best_mpu = mpu;
        best_ks = ks_run;
        best_runs = 1;
      }
  }
  for (int mpu = 1; mpu <= mpu_max && !best_mpu; ++mpu)
    for (int ko = 0; ko < 4 && !best_mpu; ++ko)
      if (fits(0, ks_opts[ko], mpu) && forced_ok(0, ks_opts[ko], mpu)) {
        best_mpu = mpu;
        best_ks = ks_opts[ko];
      }
  VM_REQUIRE(best_mpu > 0, VM_E_UNSUPPORTED, "vm_conv3d_wgrad_tc: no stage configuration fits");
  p.mt_per_unit = best_mpu;
  p.KS = best_ks;
  p.runs = best_runs;
  p.RR = p.KS + 8;
  p.runs_alloc = (16 * p.mt_per_unit + 2) / 3 + 2;
  // TMA tensor destinations (the gy box) must be 128-byte aligned: keep every region 1 KB aligned
  p.a_bytes = ((p.runs ? (uint32_t)p.runs_alloc * 3 * p.Wp * 16 : (uint32_t)p.mt_per_unit * 16 * p.RR * 16) + 1023) & ~1023u;
  p.g_bytes = (uint32_t)p.CGo * p.RR * 16;
  p.stage_bytes = (p.a_bytes + g_region(p.KS) + 1023) & ~1023u;
  p.stages = kSmemBudget / (int)p.stage_bytes;
  if (p.stages > kMaxStages) p.stages = kMaxStages;
  VM_REQUIRE(p.stages >= 2 && p.mt_per_unit >= 1, VM_E_UNSUPPORTED, "vm_conv3d_wgrad_tc: stage does not fit");
  p.n_mtgroups = (p.MT + p.mt_per_unit - 1) / p.mt_per_unit;
  const int64_t anchors = (int64_t)D * p.P;
  p.stages_total = (int)((anchors + p.KS - 1) / p.KS);
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  // one unit per CTA (a second wave of units would double the slowest CTA's time): as many
  // K splits as fit in one wave, at least g_wg_min_spk stages per unit (pipeline fill)
  const int ncol = p.n_mtgroups * p.nchunk;
  int want = nsm / (ncol * B);
  if (want < 1) want = 1;
  p.spk = (p.stages_total + want - 1) / want;
  if (p.spk < g_wg_min_spk) p.spk = g_wg_min_spk;
  p.ksplit = (p.stages_total + p.spk - 1) / p.spk;
  p.units = ncol * B * p.ksplit;
  // (interleaved: 64->64 at 128^3 547 -> 535 us, 192->64 1281 -> 1242 us, 64->64 at 32^3 +2%)
  p.kinter = g_wg_interleave != 0;
  p.idesc = make_idesc_bf16(128, p.Nc, true, true);
  p.grid = p.units;
  if (p.grid > nsm) p.grid = (nsm / ncol) * ncol;  // CTA keeps one (chunk, M-tile group) column
  if (p.grid < ncol) p.grid = ncol;
  pl.ws_main = (size_t)(p.grid / ncol) * p.MT * 3 * p.NcTot * 128 * sizeof(float);
  pl.ws_bias = p.ones_slot >= 0 ? 0 : bias_grad_ws_bytes((int64_t)B * D * H * W, Cout);
  return VM_OK;
}

// 4-D gy map with 128-byte inner boxes: (64 = 8 rows x 8 ch, rows/8, CG, B)
// rows: rows addressable from `base` (later rows read as zeros), stride_rows: rows between
// channel-group planes
int make_wide_map(CUtensorMap* m, const void* base, int64_t bstride, int CG, int64_t rows, int64_t stride_rows,
                  int B, int box_blocks, int box_groups) {
  auto enc = encode_fn();
  VM_REQUIRE(enc, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  VM_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, VM_E_ALIGN, "slab base not 16B aligned");
  cuuint64_t dims[4] = {64, (cuuint64_t)(rows / 8), (cuuint64_t)CG, (cuuint64_t)B};
  cuuint64_t strides[3] = {128, (cuuint64_t)stride_rows * 16, (cuuint64_t)bstride * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_blocks, (cuuint32_t)box_groups, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  VM_REQUIRE(r == CUDA_SUCCESS, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled (wide) failed (%d)", (int)r);
  return VM_OK;
}

int make_group_map(CUtensorMap* m, const void* base, int64_t bstride, int CG, int64_t rows, int64_t stride_rows,
                   int B, int box_rows, int box_groups) {
  auto enc = encode_fn();
  VM_REQUIRE(enc, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {8, (cuuint64_t)rows, (cuuint64_t)CG, (cuuint64_t)B};
  cuuint64_t strides[3] = {16, (cuuint64_t)stride_rows * 16, (cuuint64_t)bstride * 2};
  cuuint32_t box[4] = {8, (cuuint32_t)box_rows, (cuuint32_t)box_groups, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  VM_REQUIRE(r == CUDA_SUCCESS, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled (group) failed (%d)", (int)r);
  return VM_OK;
}
}  // namespace


static int g_skip_wg_fin = 0;
extern "C" void vm_debug_skip_wgrad_finalize(int v) { g_skip_wg_fin = v; }
extern "C" void vm_debug_set_wgrad_kd_runtime(int v) { g_wk_runtime = v; }
extern "C" void vm_debug_set_wgrad_interleave(int v) { g_wg_interleave = v; }
extern "C" void vm_debug_set_wgrad_chunk(int v) { g_wg_chunk = v; }
extern "C" void vm_debug_set_wgrad_merge(int v) { g_wg_merge = v; }
extern "C" void vm_debug_set_wgrad_ksub_stages(int v) { g_wk_ksub_min_stages = v > 0 ? v : 2; }

extern "C" void vm_debug_set_wgrad_min_spk(int v) { g_wg_min_spk = v > 0 ? v : 2; }

extern "C" void vm_debug_force_wgrad_plan(int runs, int ks, int mpu) {
  g_force_runs = runs;
  g_force_ks = ks;
  g_force_mpu = mpu;
}

extern "C" int vm_debug_wgrad_plan(int B, int Cin, int Cout, int D, int H, int W, int* out) {
  WgPlan pl;
  int rc = plan_wgrad(B, Cin, Cout, D, H, W, pl);
  if (rc) return rc;
  const WgParams& p = pl.p;
  const int v[12] = {p.runs, p.KS, p.MT, p.mt_per_unit, p.n_mtgroups, p.stages, p.ksplit, p.spk,
                     p.units, p.ones_slot, (int)p.stage_bytes, p.gdelta};
  for (int i = 0; i < 12; ++i) out[i] = v[i];
  return VM_OK;
}

// Plan of the kd-along-N weight-gradient kernel; false when the shape is not eligible
// (3*Nc > 144 or TMEM, rows narrower than 34, or no double-buffered stage fits).
static bool plan_wgrad_kd(int B, int Cin, int Cout, int D, int H, int W, WkParams& p, size_t& ws) {
  p = WkParams{};
  if (g_force_runs == 0 || g_force_runs == 2) return false;  // debug override: the general kernel
  p.B = B;
  p.Wp = W + 2;
  p.P = (H + 2) * p.Wp;
  p.rows = (D + 2) * p.P;
  p.plane8 = (int64_t)p.rows * 8;
  p.CG = (Cin + 7) / 8;
  p.CGo = (Cout + 7) / 8;
  p.Cout = Cout;
  p.Nc = (Cout + 15) / 16 * 16;
  if (3 * p.Nc > 256) return false;  // N = 3*Nc per MMA
  p.KS = min(256, ((p.Wp - 2) / 16) * 16);  // a run of KS + 2Wp + 2 rows fits 3 slots of Wp rows
  if (p.KS < 32) return false;
  // Nc > 48 needs one kw tap per CTA, which triples the A traffic per output: the general
  // kernel wins at every such shape measured (tools/dbg_wgrad_modes.py: 64->64 at 128^3
  // 0.55 vs 0.98 ms, 192->64 1.28 vs 4.75 ms, 32->64 0.38 vs 0.84 ms, 16->80 at 64^3
  // 0.054 vs 0.12 ms), while Cout <= 48 stays here (32->32 at 256^3: 1.19 vs 3.50 ms)
  if (p.Nc > 48) return false;
  if ((3 * p.CG) % 16 == 0) return false;  // no spare M slot for the bias-gradient ones block
  p.MT = (3 * p.CG + 1 + 15) / 16;
  p.ones_slot = 3 * p.CG;
  // TMEM: mt_per_unit tiles x nkw kw accumulators x 3*Nc columns <= 512
  p.nkw = 9 * p.Nc <= 512 ? 3 : 1;
  p.mt_per_unit = 512 / (p.nkw * 3 * p.Nc);
  if (p.mt_per_unit > p.MT) p.mt_per_unit = p.MT;
  if (g_force_mpu > 0 && g_force_mpu < p.mt_per_unit) p.mt_per_unit = g_force_mpu;  // A/B probes
  while (p.mt_per_unit > 1 && p.MT % p.mt_per_unit) --p.mt_per_unit;  // equal groups (kernel template)
  if (p.mt_per_unit < 1) return false;
  if (g_force_ks >= 32 && g_force_ks % 16 == 0 && g_force_ks < p.KS) p.KS = g_force_ks;  // A/B probes
  for (;;) {
    p.g_bytes = (uint32_t)(p.Nc / 8) * p.KS * 16;
    p.g_load = (uint32_t)p.CGo * p.KS * 16;
    // slot positions a CTA touches: its 16*mt_per_unit M slots (+ up to 2 of run alignment),
    // never more than the 3*CG run slots + the ones slot; + 1 slot of slack for the last run
    const int slots = min(16 * p.mt_per_unit + 2, 3 * p.CG + 1) + 1;
    p.a_bytes = ((uint32_t)slots * p.Wp * 16 + 1023) & ~1023u;
    p.sub_bytes = (p.a_bytes + 3 * p.g_bytes + 1023) & ~1023u;
    // two K chunks per stage halve the per-stage MMA-warp bookkeeping when 4 stages still fit
    p.ksub = kSmemBudget / (int)(2 * p.sub_bytes) >= g_wk_ksub_min_stages ? 2 : 1;
    p.stage_bytes = p.ksub * p.sub_bytes;
    p.stages = kSmemBudget / (int)p.stage_bytes;
    if (p.stages >= 2) break;
    if (p.mt_per_unit > 1) {
      do --p.mt_per_unit; while (p.mt_per_unit > 1 && p.MT % p.mt_per_unit);
      continue;
    }
    // one M-tile per CTA and still no double buffer (wide rows x many input channel groups,
    // e.g. the decoder's 96 -> 32 conv at 256^3): shorter K chunks shrink the gy slices
    if (p.KS <= 32) break;
    p.KS = max(32, (p.KS / 2) / 16 * 16);
  }
  if (p.stages < 2) return false;
  if (p.stages > kMaxStages) p.stages = kMaxStages;
  p.n_mtgroups = (p.MT + p.mt_per_unit - 1) / p.mt_per_unit;
  p.ngroups = p.n_mtgroups * (3 / p.nkw);
  p.stages_total = (p.rows + p.KS * p.ksub - 1) / (p.KS * p.ksub);
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  int want = (2 * nsm + p.ngroups * B - 1) / (p.ngroups * B);  // ~2 units per SM
  if (want < 1) want = 1;
  p.spk = (p.stages_total + want - 1) / want;
  if (p.spk < 2) p.spk = 2;
  p.ksplit = (p.stages_total + p.spk - 1) / p.spk;
  p.units = p.ngroups * B * p.ksplit;
  // interleaved stages (tools/wgrad_inter_ab.py, alternating A/B, best of 3): 32->32 at 256^3
  // 1159 -> 1096 us, 48->16 / 32->32 at 64^3 neutral to +1%; with several M-tile groups (96->32
  // at 256^3) the groups' CTAs of one stage are no longer co-scheduled: 5388 -> 5507 us
  p.kinter = g_wg_interleave == 2 || (g_wg_interleave == 1 && p.ngroups == 1);
  p.idesc = make_idesc_bf16(128, 3 * p.Nc, true, true);
  p.idesc64 = make_idesc_bf16(64, 3 * p.Nc, true, true);
  p.grid = p.units;
  if (p.grid > nsm) p.grid = (nsm / p.ngroups) * p.ngroups;
  if (p.grid < p.ngroups) p.grid = p.ngroups;
  ws = (size_t)(p.grid / p.ngroups) * p.MT * 9 * p.Nc * 128 * sizeof(float);
  return true;
}

// Output channels per weight-gradient call: the accumulators of one M-tile are 3 kw x Nc
// TMEM columns (<= 512), so wider layers (cfg3/cfg4: up to 512 -> 1024 channels) run as
// chunks of 128 output channels; each chunk reads its own channel-group planes of gy.

// Input-channel chunks of the kd weight gradient: a layer whose (cg, kh) slots span several
// M-tile groups (the decoder's concat convs, 96->32) runs as chunks of 32 input channels, one
// M-tile each (13 of 16 slots live, 256-anchor K chunks), writing its rows of gw in place
// (one call: 3 M-tile groups, 5 live slots in the third tile, shorter K chunks to fit)
constexpr int kWgChunkCin = 32;
// (tools/wgrad_chunk_ab.py, alternating A/B: 96->32 at 256^3 5.41 -> 3.30 ms, 64->32 at 256^3
// 2.68 -> 2.22 ms; at 2 M voxels only three or more chunks win: 96->32 at 32x256x256 (a depth-
// split rank's block of 256^3) 678 -> 467 us, 96->32 at 128^3 1.08x, 64->32 at 128^3 0.90x,
// 96->32 at 64x128x128 0.82x)
static bool wgrad_kd_chunked(int B, int Cin, int Cout, int D, int H, int W) {
  WkParams pk;
  size_t wsk = 0;
  const int64_t vox = (int64_t)B * D * H * W;
  return (g_wg_chunk == 2 || vox >= (1 << 22) || (vox >= (1 << 21) && Cin >= 3 * kWgChunkCin)) &&
         Cin > kWgChunkCin && Cin % kWgChunkCin == 0 &&
         plan_wgrad_kd(B, Cin, Cout, D, H, W, pk, wsk) &&
         pk.ngroups > 1 && plan_wgrad_kd(B, kWgChunkCin, Cout, D, H, W, pk, wsk);
}

extern "C" size_t vm_conv3d_wgrad_tc_ws(int B, int Cin, int Cout, int D, int H, int W) {
  if (Cout > kWgradMaxCout && !wgrad_merged_chunks(Cout)) Cout = kWgradChunk;  // one call per chunk: the widest
  WkParams pk;
  size_t wsk = 0;
  if (plan_wgrad_kd(B, Cin, Cout, D, H, W, pk, wsk)) {
    size_t wsc = 0;
    if (wgrad_kd_chunked(B, Cin, Cout, D, H, W)) plan_wgrad_kd(B, kWgChunkCin, Cout, D, H, W, pk, wsc);
    return (wsk > wsc ? wsk : wsc) + 256;
  }
  WgPlan pl;
  if (plan_wgrad(B, Cin, Cout, D, H, W, pl) != VM_OK) return 0;
  return pl.ws_main + pl.ws_bias + 256;
}

// One call of the weight-gradient kernels for Cout <= kWgradMaxCout output channels; gw rows
// have stride ldo (>= Cout) so that a chunk of a wider layer writes its columns in place.
static int wgrad_tc_one(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride, float* gw, float* gb,
                        void* ws, int B, int Cin, int Cout, int D, int H, int W, int ldo, void* stream,
                        int ci_stride = 0) {
  if (ci_stride <= 0) ci_stride = Cin;
  if (ci_stride == Cin && g_wg_chunk && wgrad_kd_chunked(B, Cin, Cout, D, H, W)) {
    const int64_t xbs = x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1);
    const int64_t plane8 = (int64_t)(D + 2) * (H + 2) * (W + 2) * 8;
    for (int c0 = 0; c0 < Cin; c0 += kWgChunkCin) {
      const int rc = wgrad_tc_one(static_cast<const bf16*>(x) + (int64_t)(c0 / 8) * plane8, xbs, gy, gy_bstride,
                                  gw + (int64_t)c0 * ldo, c0 == 0 ? gb : nullptr, ws, B, kWgChunkCin, Cout, D, H, W,
                                  ldo, stream, Cin);
      if (rc) return rc;
    }
    return VM_OK;
  }
  {
    WkParams pk;
    size_t wsk = 0;
    if (plan_wgrad_kd(B, Cin, Cout, D, H, W, pk, wsk)) {
      pk.x = static_cast<const bf16*>(x);
      pk.x_bstride = x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1);
      pk.ws = static_cast<float*>(ws);
      pk.dbg = g_fwd_dbg;
      const int64_t gbs = gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1);
      CUtensorMap gmap;
      // gy through its interior depth planes only (rows [P, (D+1)P) from the plane-1 base): the
      // depth margin layers read as zeros even while a halo exchange is filling them, so the
      // weight gradient can run concurrently with the output gradient's exchange + dgrad
      int rc = make_group_map(&gmap, static_cast<const bf16*>(gy) + (int64_t)pk.P * 8, gbs, pk.CGo,
                              (int64_t)D * pk.P, pk.rows, B, pk.KS, pk.CGo);
      if (rc) return rc;
      cudaStream_t st = as_stream(stream);
      const bool dbg = pk.dbg != nullptr;
      const int phase = g_wg_phase;
      using WkKern = void (*)(const CUtensorMap, const WkParams);
      // [NMT-1][variant]: 0 runtime, then (NKK, KSUB) = (2,1) (2,2) (4,1) (4,2) (8,1) (8,2) (16,1) (16,2)
#define WK_ROW(M)                                                                                               \
  {k_conv_wgrad_kd<M, 0, 0>, k_conv_wgrad_kd<M, 2, 1>,  k_conv_wgrad_kd<M, 2, 2>, k_conv_wgrad_kd<M, 4, 1>,     \
   k_conv_wgrad_kd<M, 4, 2>, k_conv_wgrad_kd<M, 8, 1>,  k_conv_wgrad_kd<M, 8, 2>, k_conv_wgrad_kd<M, 16, 1>,    \
   k_conv_wgrad_kd<M, 16, 2>}
      static const WkKern table[3][9] = {WK_ROW(1), WK_ROW(2), WK_ROW(3)};
#undef WK_ROW
      const int nkk = pk.KS / 16;
      int var = 0;
      if (pk.nkw == 3 && (pk.ksub == 1 || pk.ksub == 2) && (nkk == 2 || nkk == 4 || nkk == 8 || nkk == 16) &&
          !g_wk_runtime)
        var = (nkk == 2 ? 1 : nkk == 4 ? 3 : nkk == 8 ? 5 : 7) + (pk.ksub - 1);
      auto kern = table[pk.mt_per_unit - 1][var];
      (void)dbg;
      if (phase != 2) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
        launch_pdl(kern, pk.grid, 192, (size_t)pk.stages * pk.stage_bytes, st, gmap, pk);
        rc = launch_status("vm_conv3d_wgrad_tc (kd)");
        if (rc) return rc;
      }
      if (phase == 1) return VM_OK;  // the finalize is issued separately (vm_conv3d_wgrad_tc_phase)
      const int nk = pk.grid / pk.ngroups;
      const int ntiles = pk.MT * 3 * (3 * pk.Nc / 8) * 4;
      // many partials (one per CTA of a wide K split): 32 warps per tile keep more loads in flight
      auto fin = nk >= 64 ? k_wgrad_finalize_tiles<true, 32> : k_wgrad_finalize_tiles<true, 8>;
      if (g_skip_wg_fin) return VM_OK;  // A/B probe (wrong results): the finalize's share of a step
      launch_pdl(fin, ntiles, nk >= 64 ? 1024 : 256, 0, st, pk.ws, gw, gb, nk, pk.MT, pk.Nc, pk.CG, Cin, Cout,
                                                          pk.ones_slot, 0, nullptr, 0, 0, Cout, ci_stride);
      return launch_status("vm_conv3d_wgrad_tc (kd) finalize");
    }
  }
  WgPlan pl;
  int rc = plan_wgrad(B, Cin, Cout, D, H, W, pl);
  if (rc) return rc;
  WgParams p = pl.p;
  p.x = static_cast<const bf16*>(x);
  p.x_bstride = x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1);
  p.ws = static_cast<float*>(ws);
  p.dbg = g_fwd_dbg;
  const int64_t gbs = gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1);
  const int64_t rows = (int64_t)(D + 2) * p.P;
  CUtensorMap gmap;
  // anchors never reach gy's margin layer 0; its margin layer D+1 (exchanged concurrently, see
  // the kd kernel) is cut off: rows >= (D+1)P read as zeros (the wide map's 8-row blocks round
  // down: the < 8 rows dropped lie in layer D's h = H+1 margin row, zero, as W + 2 >= 8 there)
  int64_t glim = rows - p.P;
  if (p.gwide && glim % 8 > p.Wp) glim += 8 - glim % 8;  // never drop interior rows (W + 2 < 8)
  const int cgo_all = p.nchunk * p.CGo;
  rc = p.gwide ? make_wide_map(&gmap, gy, gbs, cgo_all, glim, rows, B, p.RR / 8, p.CGo)
               : make_group_map(&gmap, gy, gbs, cgo_all, glim, rows, B, p.RR, p.CGo);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  // compile-time M-tile count (when every CTA holds the same number of tiles) and K steps
  const bool even = p.MT % p.mt_per_unit == 0;
  const int nmt_t = even && p.mt_per_unit <= 4 ? p.mt_per_unit : 0;
  const int nkk_t = (p.KS == 64 || p.KS == 128 || p.KS == 192 || p.KS == 256) ? p.KS / 16 : 0;
  using WgKern = void (*)(const CUtensorMap, const WgParams);
  static const WgKern table[5][5] = {
      {k_conv_wgrad_tc<0, 0>, k_conv_wgrad_tc<0, 4>, k_conv_wgrad_tc<0, 8>, k_conv_wgrad_tc<0, 12>, k_conv_wgrad_tc<0, 16>},
      {k_conv_wgrad_tc<1, 0>, k_conv_wgrad_tc<1, 4>, k_conv_wgrad_tc<1, 8>, k_conv_wgrad_tc<1, 12>, k_conv_wgrad_tc<1, 16>},
      {k_conv_wgrad_tc<2, 0>, k_conv_wgrad_tc<2, 4>, k_conv_wgrad_tc<2, 8>, k_conv_wgrad_tc<2, 12>, k_conv_wgrad_tc<2, 16>},
      {k_conv_wgrad_tc<3, 0>, k_conv_wgrad_tc<3, 4>, k_conv_wgrad_tc<3, 8>, k_conv_wgrad_tc<3, 12>, k_conv_wgrad_tc<3, 16>},
      {k_conv_wgrad_tc<4, 0>, k_conv_wgrad_tc<4, 4>, k_conv_wgrad_tc<4, 8>, k_conv_wgrad_tc<4, 12>, k_conv_wgrad_tc<4, 16>},
  };
  auto kern = table[nmt_t][nkk_t / 4];
  const int phase = g_wg_phase;
  if (phase != 2) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    launch_pdl(kern, p.grid, 192, (size_t)p.stages * p.stage_bytes, st, gmap, p);
    rc = launch_status("vm_conv3d_wgrad_tc");
    if (rc) return rc;
  }
  const int nk = p.grid / (p.n_mtgroups * p.nchunk);
  // without a ones slot the bias gradient comes from separate partials, reduced by the
  // finalize's extra blocks
  int nsb = 0;
  float* wsb = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ((pl.ws_main + 255) / 256) * 256);
  if (p.ones_slot < 0) {
    if (phase != 2) {
      rc = bias_grad_partial_bf16(gy, gbs, wsb, B, Cout, D, H, W, st, &nsb);
      if (rc) return rc;
    } else {
      nsb = bias_grad_partial_count(B, Cout, D, H, W);
    }
  }
  if (phase == 1) return VM_OK;
  const int ntiles = p.MT * 3 * (p.NcTot / 8) * 4;
  const int nbias = p.ones_slot < 0 ? (Cout + 255) / 256 : 0;
  if (g_skip_wg_fin) return VM_OK;
  launch_pdl(k_wgrad_finalize_tiles<false, 8>, ntiles + nbias, 256, 0, st, p.ws, gw, gb, nk, p.MT, p.NcTot, p.CG, Cin, Cout,
                                                               p.ones_slot, p.runs, wsb, nsb, (Cout + 7) / 8, ldo, ci_stride);
  return launch_status("vm_conv3d_wgrad_tc finalize");
}

// The weight gradient in two stream-ordered halves, so that the K-split finalize of one layer
// can run on another stream while the next layer's main kernel starts (the caller alternates
// two workspaces): phase 1 launches the main kernel (and the bias partials), phase 2 the
// finalize of the same call's workspace.  Layers that run as several calls into one workspace
// (output-channel chunks, input-channel chunks) do everything in phase 1; phase 2 is a no-op.
extern "C" int vm_conv3d_wgrad_tc_deferrable(int B, int Cin, int Cout, int D, int H, int W) {
  return (Cout <= kWgradMaxCout || wgrad_merged_chunks(Cout)) && !wgrad_kd_chunked(B, Cin, Cout, D, H, W);
}
extern "C" int vm_conv3d_wgrad_tc_phase(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride,
                                        float* gw, float* gb, void* ws, int B, int Cin, int Cout, int D, int H,
                                        int W, int phase, void* stream) {
  VM_REQUIRE(phase >= 0 && phase <= 2, VM_E_ARG, "vm_conv3d_wgrad_tc_phase: phase %d", phase);
  const bool split = phase != 0 && vm_conv3d_wgrad_tc_deferrable(B, Cin, Cout, D, H, W);
  if (phase == 2 && !split) return VM_OK;
  g_wg_phase = split ? phase : 0;
  const int rc = vm_conv3d_wgrad_tc(x, x_bstride, gy, gy_bstride, gw, gb, ws, B, Cin, Cout, D, H, W, stream);
  g_wg_phase = 0;
  return rc;
}

extern "C" int vm_conv3d_wgrad_tc(const void* x, int64_t x_bstride, const void* gy,
                                  int64_t gy_bstride, float* gw, float* gb, void* ws, int B, int Cin,
                                  int Cout, int D, int H, int W, void* stream) {
  VM_REQUIRE(x && gy && gw && gb && ws, VM_E_ARG, "vm_conv3d_wgrad_tc: null pointer");
  VM_REQUIRE(B > 0 && Cin > 0 && Cout > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE,
             "vm_conv3d_wgrad_tc: bad shape");
  const int64_t gbs = gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1);
  if (Cout <= kWgradMaxCout || wgrad_merged_chunks(Cout))
    return wgrad_tc_one(x, x_bstride, gy, gbs, gw, gb, ws, B, Cin, Cout, D, H, W, Cout, stream);
  const int64_t plane8 = (int64_t)(D + 2) * (H + 2) * (W + 2) * 8;
  for (int co0 = 0; co0 < Cout; co0 += kWgradChunk) {
    const int cc = min(kWgradChunk, Cout - co0);
    const bf16* gyc = static_cast<const bf16*>(gy) + (int64_t)(co0 / 8) * plane8;
    const int rc = wgrad_tc_one(x, x_bstride, gyc, gbs, gw + co0, gb + co0, ws, B, Cin, cc, D, H, W, Cout, stream);
    if (rc) return rc;
  }
  return VM_OK;
}
