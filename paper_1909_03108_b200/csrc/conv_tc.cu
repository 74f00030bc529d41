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
constexpr bool kFoldEnabled = false;

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
// Packed forward operand: [nchunk][kc][kd][9 taps (kh,kw)][2 K-halves][Nc][8] bf16, where
// ci = (kc*2 + half)*8 + e, co = nchunk*Nc + n.  flip = 1 packs the dgrad operand:
// W'[t'][ci'][co'] = W[26 - t'][co'][ci'] (conv of the output gradient).
struct PackGeom {
  int cin, cout;   // of the conv this operand feeds
  int CG, KC;      // input channel groups, chunks of 2 groups
  int Nc, nchunk;  // N per chunk (multiple of 16, <= 256)
  int fold;        // thin output (Nc <= 32): kw folded into N, layout [kc][kd][kh][2][3*Nc][8]
};

__host__ __device__ static PackGeom pack_geom(int cin, int cout) {
  PackGeom g;
  g.cin = cin;
  g.cout = cout;
  g.CG = (cin + 7) / 8;
  g.KC = (g.CG + 1) / 2;
  int npad = (cout + 15) / 16 * 16;
  g.nchunk = (npad + 255) / 256;
  g.Nc = ((npad + g.nchunk - 1) / g.nchunk + 15) / 16 * 16;
  // kw-folded kernel (k_conv_fwd_fold): correct, but on B200 its shift-add epilogue is
  // CUDA-core bound (~10 instr / output) and loses to the plain kernel; kept, not selected.
  g.fold = (kFoldEnabled && g.nchunk == 1 && g.Nc <= 32) ? 1 : 0;
  return g;
}

// Value of packed element `r` (see PackGeom for the two layouts).  flip = 1 packs the dgrad
// operand W'[t'][ci'][co'] = W[26 - t'][co'][ci'].
__device__ __forceinline__ float pack_value(const PackGeom& g, int64_t r, const float* __restrict__ w,
                                            int layer_cin, int layer_cout, int flip) {
  const int e = r % 8;
  r /= 8;
  int kd, kh, kw, kc, nch, co, half;
  if (g.fold) {
    const int n = r % (3 * g.Nc);
    r /= 3 * g.Nc;
    half = r % 2;
    r /= 2;
    kh = r % 3;
    r /= 3;
    kd = r % 3;
    kc = (int)(r / 3);
    kw = n / g.Nc;
    co = n % g.Nc;
    nch = 0;
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
    nch = (int)(r / g.KC);
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
  int mblocks;       // per sample
  int units;
  uint32_t a_bytes;  // per group per stage
  uint32_t b_bytes;  // per stage
  uint32_t stage_bytes;
  uint32_t idesc;
  unsigned flags;
  long long* dbg;  // optional timing probes [gridDim][4]
  int TS;          // anchors between consecutive tiles (128; 126 in the kw-folded kernel)
  uint32_t wp_magic, hp_magic;  // floor(2^32 / d) + 1 for the anchor (w, h) split
};

__global__ void __launch_bounds__(320, 1)
    k_conv_fwd_tc(const FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ float sbias[1024];
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
  const int nstage_k = p.KC * 3;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int nch = u % p.nchunk;
        const int mb = (u / p.nchunk) % p.mblocks;
        const int b = u / (p.nchunk * p.mblocks);
        const int64_t a0 = (int64_t)mb * p.MB * 128;
        for (int kc = 0; kc < p.KC; ++kc) {
          const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
          for (int kd = 0; kd < 3; ++kd) {
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
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    long long t_wait_tmem = 0, t_wait_full = 0, t_start = clock64();
    int stage = 0;
    uint32_t phase = 0;
    int ab = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      long long tw0 = clock64();
      mbar_wait(&tempty[ab], aphase ^ 1);
      t_wait_tmem += clock64() - tw0;
      tc_fence_after();
      for (int s = 0; s < nstage_k; ++s) {
        const int kc = s / 3;
        const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
        long long tf0 = clock64();
        mbar_wait(&full[stage], phase);
        t_wait_full += clock64() - tf0;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sB = sA + 2 * p.a_bytes;
          const uint32_t lbo_a = ng == 2 ? p.a_bytes : 0;
          // descriptors advance by plain adds on the 16-byte address field
          const uint64_t a0desc = make_sdesc(sA, lbo_a, 128);
          const uint64_t b0desc = make_sdesc(sB, p.Nc * 16, 128);
          const uint32_t d0 = tbase + (uint32_t)(ab * p.MB * p.Nc);
          const uint32_t bstep = (uint32_t)(2 * p.Nc * 16) >> 4;
#pragma unroll 1
          for (int j = 0; j < 9; ++j) {
            const uint64_t bdesc = b0desc + (uint64_t)(j * bstep);
            const uint64_t adesc = a0desc + (uint64_t)((j / 3) * p.Wp + (j % 3));
            const uint32_t acc = (s > 0 || j > 0) ? 1u : 0u;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < p.MB)
                mma_bf16_ss(d0 + (uint32_t)(i * p.Nc), adesc + (uint64_t)(i * 128), bdesc, p.idesc, acc);
            }
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
      if (++ab == 2) {
        ab = 0;
        aphase ^= 1;
      }
    }
    if (p.dbg && lane == 0) {
      p.dbg[blockIdx.x * 4 + 0] = clock64() - t_start;
      p.dbg[blockIdx.x * 4 + 1] = t_wait_tmem;
      p.dbg[blockIdx.x * 4 + 2] = t_wait_full;
    }
  } else {
    // ===================== epilogue (warps 2..9) =====================
    // warp w drains TMEM lane quarter (w & 3) of every other tile (parity (w-2)/4)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;  // 0..255
    if (!(p.flags & VM_CONV_NOBIAS))
      for (int c = et; c < p.Cout; c += 256) sbias[c] = p.bias[c];
    asm volatile("bar.sync 1, 256;" ::: "memory");
    int ab = 0;
    uint32_t aphase = 0;
    long long t_epi_wait = 0;
    const int ng_out = p.Nc / 8;
    const bool domask = p.flags & VM_CONV_MASK;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int nch = u % p.nchunk;
      const int mb = (u / p.nchunk) % p.mblocks;
      const int b = u / (p.nchunk * p.mblocks);
      const int a0 = mb * p.MB * 128;
      const bf16* mbase = p.mask + b * p.m_bstride;
      bf16* ybase = p.y + b * p.y_bstride;
      long long te0 = clock64();
      mbar_wait(&tfull[ab], aphase);
      t_epi_wait += clock64() - te0;
      tc_fence_after();
      for (int i = half; i < p.MB; i += 2) {
        const int a = a0 + i * 128 + q * 32 + lane;
        // (w, h) of the anchor via multiply-high division (divisors are small)
        uint32_t qa = __umulhi((uint32_t)a, p.wp_magic);
        if (qa * (uint32_t)p.Wp > (uint32_t)a) --qa;
        if ((qa + 1) * (uint32_t)p.Wp <= (uint32_t)a) ++qa;
        const int wq = a - (int)qa * p.Wp;
        uint32_t qh = __umulhi(qa, p.hp_magic);
        if (qh * (uint32_t)p.Hp > qa) --qh;
        if ((qh + 1) * (uint32_t)p.Hp <= qa) ++qh;
        const int hq = (int)qa - (int)qh * p.Hp;
        const bool valid = a < p.anchors && wq < p.W && hq < p.H;
        const int64_t orow = (int64_t)a + p.P + p.Wp + 1;
        const uint32_t tcol = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * p.MB + i) * p.Nc);
        for (int g0 = 0; g0 < ng_out; g0 += 8) {
          const int gn = min(8, ng_out - g0);
          int4 mk[8];
          if (domask) {  // issue the mask loads first (latency overlap)
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
            uint32_t r[16];
            if (j + 1 < gn) {
              tmem_ld16(tcol + (uint32_t)((g0 + j) * 8), r);
            } else {
              uint32_t r8[8];
              tmem_ld8(tcol + (uint32_t)((g0 + j) * 8), r8);
#pragma unroll
              for (int e = 0; e < 8; ++e) r[e] = r8[e];
            }
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              if (j + jj >= gn) break;
              const int co0 = nch * p.Nc + (g0 + j + jj) * 8;
              if (!valid || co0 >= p.Cout) continue;
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                v[e] = __uint_as_float(r[jj * 8 + e]);
                if (!(p.flags & VM_CONV_NOBIAS)) v[e] += (co0 + e < p.Cout) ? sbias[co0 + e] : 0.f;
              }
              if (p.flags & VM_CONV_RELU) {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
              }
              if (domask) {
                const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&mk[j + jj]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  float2 f = __bfloat1622float2(mh[e]);
                  if (!(f.x > 0.f)) v[2 * e] = 0.f;
                  if (!(f.y > 0.f)) v[2 * e + 1] = 0.f;
                }
              }
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (co0 + e >= p.Cout) v[e] = 0.f;
              int4 out;
              __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
              for (int e = 0; e < 4; ++e) oh[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
              *reinterpret_cast<int4*>(ybase + (co0 / 8) * p.plane8 + orow * 8) = out;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[ab]);
      if (++ab == 2) {
        ab = 0;
        aphase ^= 1;
      }
    }
    if (p.dbg && threadIdx.x == 64) p.dbg[blockIdx.x * 4 + 3] = t_epi_wait;
  }
  tc_fence_before();
  __syncthreads();
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
  int CG, CGo, Cout, Nc;
  int KS, RR;       // anchors per stage, staged rows per group (KS + 8)
  int gdelta;       // row misalignment of the gy box start (128B-inner mode)
  int gwide;        // 1: gy map has 128-byte inner boxes
  int MT, mt_per_unit, n_mtgroups;
  int ones_slot;    // absolute M slot of the ones block, -1 if none
  int runs;         // 1: stage one run of KS+2Wp+2 rows per (kd, cg) serving all three kh
                    //    (M slot g' = (kd*CG + cg)*3 + kh, slot stride Wp rows); 0: one copy per slot
  int runs_alloc;   // run slots per stage buffer (runs mode)
  int fold;         // 1: kw folded into N (B = three kw-shifted copies of gy made in SMEM)
  int RRg;          // fold mode: rows of the raw gy box (KS + 16, 8-row aligned start)
  uint32_t gc_off;  // fold mode: offset of the shifted-copy region from the gy box
  int spk;          // stages per unit (K-split chunk)
  int ksplit;       // K-split chunks per sample
  int stages_total; // per sample
  int units;
  int grid;         // CTAs (a multiple of n_mtgroups); one K partial per CTA
  int stages;       // pipeline depth
  uint32_t a_bytes; // per stage: mt_per_unit*16 slots * RR * 16
  uint32_t g_bytes; // per stage loaded: CGo * RR * 16 (allocated: Nc/8 groups)
  uint32_t stage_bytes;
  uint32_t idesc;
  float* ws;        // [kidx = b*ksplit + ks][MT][3][Nc][128]
};

__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad_tc(const __grid_constant__ CUtensorMap gmap, const WgParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], ready[kMaxStages], tfull, tempty;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int mg_cta = blockIdx.x % p.n_mtgroups;  // every unit of this CTA has the same M-tile group
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
      mbar_init(&ready[s], 128);
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
  const int ngroups_total = 9 * p.CG;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&gmap);
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
        const int ks = (u / p.n_mtgroups) % p.ksplit;
        const int b = u / (p.n_mtgroups * p.ksplit);
        const int s0 = ks * p.spk, s1 = min(p.stages_total, s0 + p.spk);
        const bf16* xb = p.x + b * p.x_bstride;
        for (int s = s0; s < s1; ++s) {
          const int64_t k0 = (int64_t)s * p.KS;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + (size_t)stage * p.stage_bytes;
          uint8_t* sG = sA + p.a_bytes;
          mbar_arrive_expect_tx(&full[stage], tx);
          const int gr0 = (int)(k0 + p.P + p.Wp + 1);
          if (p.fold)
            tma_load_4d(sG, &gmap, &full[stage], 0, (gr0 - 2) >> 3, 0, b);
          else if (p.gwide)
            tma_load_4d(sG, &gmap, &full[stage], 0, (gr0 - p.gdelta) >> 3, 0, b);
          else
            tma_load_4d(sG, &gmap, &full[stage], 0, gr0, 0, b);
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
    }
  } else if (warp == 1) {
    // All units of this CTA share the M-tile group and cover disjoint K ranges: accumulate
    // them in TMEM and drain once (one partial per CTA instead of one per unit).
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sbo = GS;
    bool started = false;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int ks = (u / p.n_mtgroups) % p.ksplit;
      const int s0 = ks * p.spk, s1 = min(p.stages_total, s0 + p.spk);
      for (int s = s0; s < s1; ++s) {
        mbar_wait(p.fold ? &ready[stage] : &full[stage], phase);
        tc_fence_after();
        if (p.fold && elect_one()) {
          // kw folded into N: one MMA per (M-tile, K step), N = 3*Nc over the shifted gy copies
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sC = sA + p.a_bytes + p.gc_off;
          const uint64_t b0desc = make_sdesc(sC, 128, (uint32_t)p.KS * 16);
          const uint64_t a0desc = make_sdesc(sA + (uint32_t)slot_shift * GS, 128, sbo);
          const uint32_t mstep = 16 * (GS >> 4);
#pragma unroll 1
          for (int kk = 0; kk < p.KS / 16; ++kk) {
            const uint32_t acc = (started || kk > 0) ? 1u : 0u;
            const uint64_t bdesc = b0desc + (uint64_t)(kk * 16);
#pragma unroll 1
            for (int m = 0; m < nmt; ++m)
              mma_bf16_ss(tbase + (uint32_t)(m * 3 * p.Nc), a0desc + (uint64_t)(m * mstep + kk * 16), bdesc,
                          p.idesc, acc);
          }
          mma_commit(&empty[stage]);
        } else if (!p.fold && elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sG = sA + p.a_bytes;
          const uint64_t b0desc = make_sdesc(sG + (uint32_t)p.gdelta * 16, 128, (uint32_t)p.RR * 16);
          const uint64_t a0desc = make_sdesc(sA + (uint32_t)slot_shift * GS, 128, sbo);
          const uint32_t mstep = 16 * (GS >> 4);  // 16 slots, in 16-byte units
#pragma unroll 1
          for (int kk = 0; kk < p.KS / 16; ++kk) {
            const uint64_t bdesc = b0desc + (uint64_t)(kk * 16);
            const uint32_t acc = (started || kk > 0) ? 1u : 0u;
#pragma unroll 1
            for (int m = 0; m < nmt; ++m) {
              const uint64_t adesc = a0desc + (uint64_t)(m * mstep + kk * 16);
              const uint32_t d = tbase + (uint32_t)(m * 3 * p.Nc);
              mma_bf16_ss(d, adesc, bdesc, p.idesc, acc);
              mma_bf16_ss(d + p.Nc, adesc + 1, bdesc, p.idesc, acc);
              mma_bf16_ss(d + 2 * p.Nc, adesc + 2, bdesc, p.idesc, acc);
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
  } else {
    if (p.fold) {
      // gy shift workers: copy kw[u] = raw[u + delta - kw] for kw = 0..2, every stage
      const int et = threadIdx.x - 64;
      const int ngo = p.Nc / 8;
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int ks = (u / p.n_mtgroups) % p.ksplit;
        const int s0 = ks * p.spk, s1 = min(p.stages_total, s0 + p.spk);
        for (int s = s0; s < s1; ++s) {
          const int64_t k0 = (int64_t)s * p.KS;
          const int gr0 = (int)(k0 + p.P + p.Wp + 1);
          const int delta = gr0 - ((gr0 - 2) & ~7);
          mbar_wait(&full[stage], phase);
          const int4* raw = reinterpret_cast<const int4*>(smem + (size_t)stage * p.stage_bytes + p.a_bytes);
          int4* cp = reinterpret_cast<int4*>(smem + (size_t)stage * p.stage_bytes + p.a_bytes + p.gc_off);
          const int total = 3 * p.CGo * p.KS;
          for (int i = et; i < total; i += 128) {
            const int uu = i % p.KS;
            const int cgo = (i / p.KS) % p.CGo;
            const int kw = i / (p.KS * p.CGo);
            cp[(kw * ngo + cgo) * p.KS + uu] = raw[cgo * p.RRg + uu + delta - kw];
          }
          fence_proxy_async_smem();
          mbar_arrive(&ready[stage]);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    const int q = warp & 3;
    const int kidx = blockIdx.x / p.n_mtgroups;
    mbar_wait(&tfull, 0);
    tc_fence_after();
    const int m_row = q * 32 + lane;
    for (int m = 0; m < nmt; ++m)
      for (int kw = 0; kw < 3; ++kw)
        for (int n0 = 0; n0 < p.Nc; n0 += 16) {
          uint32_t r[16];
          tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((m * 3 + kw) * p.Nc + n0), r);
          tmem_ld_wait();
          float* dst = p.ws + ((((int64_t)kidx * p.MT + mt0 + m) * 3 + kw) * p.Nc + n0) * 128 + m_row;
#pragma unroll
          for (int e = 0; e < 16; ++e) dst[e * 128] = __uint_as_float(r[e]);
        }
    (void)tempty;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// Fixed-order reduction of the K-split partials, one thread per partial element
// (coalesced over m): ws[k][mt][kw][co][m] -> gw[t][ci][co] with t = (kd*3+kh)*3 + kw,
// g = mt*16 + m/8 = (kd*3+kh)*CG + ci/8; the ones slot (kw = 0, m%8 = 0) gives gb.
__global__ void k_wgrad_tc_finalize(const float* __restrict__ ws, float* __restrict__ gw,
                                    float* __restrict__ gb, int nk, int MT, int Nc, int CG, int Cin,
                                    int Cout, int ones_slot, int runs) {
  const int64_t E = (int64_t)MT * 3 * Nc * 128;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int m = e % 128;
    const int co = (e / 128) % Nc;
    const int kw = (e / (128 * Nc)) % 3;
    const int mt = (int)(e / (384LL * Nc));
    const int g = mt * 16 + m / 8;
    if (co >= Cout) continue;
    // slot -> (kd*3 + kh, channel group)
    const int pp = runs ? ((g / 3) / CG) * 3 + g % 3 : g / CG;
    const int cgi = runs ? (g / 3) % CG : g % CG;
    const bool is_w = g < 9 * CG && cgi * 8 + m % 8 < Cin;
    const bool is_b = g == ones_slot && kw == 0 && m % 8 == 0;
    if (!is_w && !is_b) continue;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;  // 4 independent chains, fixed order
    int k = 0;
    for (; k + 4 <= nk; k += 4) {
      s0 += ws[(k + 0) * E + e];
      s1 += ws[(k + 1) * E + e];
      s2 += ws[(k + 2) * E + e];
      s3 += ws[(k + 3) * E + e];
    }
    for (; k < nk; ++k) s0 += ws[k * E + e];
    const float s = (s0 + s1) + (s2 + s3);
    if (is_w) {
      const int ci = cgi * 8 + m % 8;
      gw[((int64_t)(pp * 3 + kw) * Cin + ci) * Cout + co] = s;
    } else {
      gb[co] = s;
    }
  }
}


// ------------------------------------------------------------------ forward, kw folded into N
// Thin outputs (Cout <= 32): the three kw taps are stacked along N (N = 3*Nc), so a tile
// needs only 9 (kd,kh) MMAs per 16 input channels instead of 27, and the kw shift moves to
// the output side: out[a] = P0[a] + P1[a+1] + P2[a+2] (P_kw = accumulator column block kw).
// Tiles of 128 anchor rows overlap by 2 (stride 126); the epilogue combines rows across TMEM
// lanes with warp shuffles plus a 3-value exchange in shared memory at warp boundaries.
__global__ void __launch_bounds__(320, 1)
    k_conv_fwd_fold(const FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ float sbias[1024];
  __shared__ float sx[2][2][4][3][32];  // [tile parity][tile-iteration parity][quarter][C1 l0, C2 l0, C2 l1][ch]
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int N3 = 3 * p.Nc;
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
  const int nstage_k = p.KC * 3;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int mb = u % p.mblocks;
        const int b = u / p.mblocks;
        const int64_t a0 = (int64_t)mb * p.MB * p.TS;
        for (int kc = 0; kc < p.KC; ++kc) {
          const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
          for (int kd = 0; kd < 3; ++kd) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = smem + (size_t)stage * p.stage_bytes;
            uint8_t* sB = sA + 2 * p.a_bytes;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)ng * p.R * 16 + p.b_bytes);
            for (int g = 0; g < ng; ++g)
              bulk_load(sA + (size_t)g * p.a_bytes,
                        p.x + b * p.x_bstride + (kc * 2 + g) * p.plane8 + (a0 + (int64_t)kd * p.P) * 8,
                        (uint32_t)p.R * 16, &full[stage]);
            bulk_load(sB, p.wpk + ((int64_t)kc * 3 + kd) * (p.b_bytes / 2), p.b_bytes, &full[stage]);
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    int ab = 0;
    uint32_t aphase = 0;
    long long t_wait_tmem = 0, t_wait_full = 0, t_start = clock64();
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      long long tw0 = clock64();
      mbar_wait(&tempty[ab], aphase ^ 1);
      t_wait_tmem += clock64() - tw0;
      tc_fence_after();
      for (int s = 0; s < nstage_k; ++s) {
        const int kc = s / 3;
        const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
        long long tf0 = clock64();
        mbar_wait(&full[stage], phase);
        t_wait_full += clock64() - tf0;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sB = sA + 2 * p.a_bytes;
          const uint64_t a0desc = make_sdesc(sA, ng == 2 ? p.a_bytes : 0, 128);
          const uint64_t b0desc = make_sdesc(sB, N3 * 16, 128);
          const uint32_t d0 = tbase + (uint32_t)(ab * p.MB * N3);
          const uint32_t bstep = (uint32_t)(2 * N3 * 16) >> 4;
#pragma unroll 1
          for (int kh = 0; kh < 3; ++kh) {
            const uint64_t bdesc = b0desc + (uint64_t)(kh * bstep);
            const uint64_t adesc = a0desc + (uint64_t)(kh * p.Wp);
            const uint32_t acc = (s > 0 || kh > 0) ? 1u : 0u;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < p.MB)
                mma_bf16_ss(d0 + (uint32_t)(i * N3), adesc + (uint64_t)(i * p.TS), bdesc, p.idesc, acc);
            }
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
      if (++ab == 2) {
        ab = 0;
        aphase ^= 1;
      }
    }
    if (p.dbg && lane == 0) {
      p.dbg[blockIdx.x * 4 + 0] = clock64() - t_start;
      p.dbg[blockIdx.x * 4 + 1] = t_wait_tmem;
      p.dbg[blockIdx.x * 4 + 2] = t_wait_full;
    }
  } else {
    // epilogue warps 2..9: warp w drains lane quarter (w & 3) of tiles with parity (w-2)/4
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;
    if (!(p.flags & VM_CONV_NOBIAS))
      for (int c = et; c < p.Cout; c += 256) sbias[c] = p.bias[c];
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const bool domask = p.flags & VM_CONV_MASK;
    const int ngo = p.Nc / 8;
    int ab = 0;
    uint32_t aphase = 0;
    int cpar = 0;
    long long e_wait = 0, e_ld = 0, e_bar = 0, e_rest = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int mb = u % p.mblocks;
      const int b = u / p.mblocks;
      const int a0 = mb * p.MB * p.TS;
      const bf16* mbase = p.mask + b * p.m_bstride;
      bf16* ybase = p.y + b * p.y_bstride;
      long long c0t = clock64();
      mbar_wait(&tfull[ab], aphase);
      e_wait += clock64() - c0t;
      tc_fence_after();
      for (int i = half; i < p.MB; i += 2) {
        long long c1t = clock64();
        const int r = q * 32 + lane;  // tile row
        const int a = a0 + i * p.TS + r;
        uint32_t qa = __umulhi((uint32_t)a, p.wp_magic);
        if (qa * (uint32_t)p.Wp > (uint32_t)a) --qa;
        if ((qa + 1) * (uint32_t)p.Wp <= (uint32_t)a) ++qa;
        const int wq = a - (int)qa * p.Wp;
        uint32_t qh = __umulhi(qa, p.hp_magic);
        if (qh * (uint32_t)p.Hp > qa) --qh;
        if ((qh + 1) * (uint32_t)p.Hp <= qa) ++qh;
        const int hq = (int)qa - (int)qh * p.Hp;
        const bool valid = r < p.TS && a < p.anchors && wq < p.W && hq < p.H;
        const int64_t orow = (int64_t)a + p.P + p.Wp + 1;
        const uint32_t tcol = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * p.MB + i) * N3);
        // whole tile at once: masks (dgrad) first, then all 3*Nc accumulator columns, one
        // exchange + barrier, then combine / store (ngo <= 4 since Nc <= 32)
        int4 mk[4];
        if (domask) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            mk[g] = (g < ngo && valid) ? __ldg(reinterpret_cast<const int4*>(mbase + g * p.plane8 + orow * 8))
                                       : make_int4(0, 0, 0, 0);
        }
        uint32_t c0[32], c1[32], c2[32];
        tmem_ld16(tcol, *reinterpret_cast<uint32_t(*)[16]>(&c0[0]));
        tmem_ld16(tcol + (uint32_t)p.Nc, *reinterpret_cast<uint32_t(*)[16]>(&c1[0]));
        tmem_ld16(tcol + (uint32_t)(2 * p.Nc), *reinterpret_cast<uint32_t(*)[16]>(&c2[0]));
        if (ngo > 2) {
          tmem_ld16(tcol + 16u, *reinterpret_cast<uint32_t(*)[16]>(&c0[16]));
          tmem_ld16(tcol + (uint32_t)(p.Nc + 16), *reinterpret_cast<uint32_t(*)[16]>(&c1[16]));
          tmem_ld16(tcol + (uint32_t)(2 * p.Nc + 16), *reinterpret_cast<uint32_t(*)[16]>(&c2[16]));
        }
        tmem_ld_wait();
        long long c2t = clock64();
        e_ld += c2t - c1t;
        float* x = &sx[half][cpar][0][0][0];  // [4 quarters][3][32]
        // lanes 0 / 1 publish the values the previous quarter's lanes 30 / 31 need (branch-free)
        {
          const bool l0 = lane == 0, l1 = lane == 1;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (e < p.Nc) {
              if (l0) x[(q * 3 + 0) * 32 + e] = __uint_as_float(c1[e]);
              if (l0) x[(q * 3 + 1) * 32 + e] = __uint_as_float(c2[e]);
              if (l1) x[(q * 3 + 2) * 32 + e] = __uint_as_float(c2[e]);
            }
          }
        }
#ifndef VM_EXPERIMENT_NOBAR
        asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
#endif
        long long c3t = clock64();
        e_bar += c3t - c2t;
        cpar ^= 1;  // next tile uses the other exchange buffer
        const int qn = q < 3 ? q + 1 : 3;
        const bool take1 = q < 3 && lane == 31, take2a = q < 3 && lane == 30, take2b = q < 3 && lane == 31;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (g >= ngo) break;
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int c = g * 8 + e;
            const float n1s = __shfl_down_sync(0xffffffffu, __uint_as_float(c1[c]), 1);
            const float n2s = __shfl_down_sync(0xffffffffu, __uint_as_float(c2[c]), 2);
            const float f1 = x[(qn * 3 + 0) * 32 + c];  // broadcast reads, no divergence
            const float f2a = x[(qn * 3 + 1) * 32 + c];
            const float f2b = x[(qn * 3 + 2) * 32 + c];
            const float n1 = take1 ? f1 : n1s;
            const float n2 = take2a ? f2a : (take2b ? f2b : n2s);
            v[e] = __uint_as_float(c0[c]) + n1 + n2;
          }
          const int co0 = g * 8;
          if (valid && co0 < p.Cout) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (!(p.flags & VM_CONV_NOBIAS)) v[e] += (co0 + e < p.Cout) ? sbias[co0 + e] : 0.f;
            if (p.flags & VM_CONV_RELU) {
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
            }
            if (domask) {
              const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&mk[g]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(mh[e]);
                if (!(f.x > 0.f)) v[2 * e] = 0.f;
                if (!(f.y > 0.f)) v[2 * e + 1] = 0.f;
              }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (co0 + e >= p.Cout) v[e] = 0.f;
            int4 out;
            __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
            for (int e = 0; e < 4; ++e) oh[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            *reinterpret_cast<int4*>(ybase + g * p.plane8 + orow * 8) = out;
          }
        }
        e_rest += clock64() - c3t;
      }
      tc_fence_before();
      mbar_arrive(&tempty[ab]);
      if (++ab == 2) {
        ab = 0;
        aphase ^= 1;
      }
    }
    if (p.dbg && threadIdx.x == 64) {
      p.dbg[4 * gridDim.x + blockIdx.x * 4 + 0] = e_wait;
      p.dbg[4 * gridDim.x + blockIdx.x * 4 + 1] = e_ld;
      p.dbg[4 * gridDim.x + blockIdx.x * 4 + 2] = e_bar;
      p.dbg[4 * gridDim.x + blockIdx.x * 4 + 3] = e_rest;
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

// Batched repack of every layer's operands in one launch (after each SGD step).
__global__ void k_pack_batch(const vm_pack_job* __restrict__ jobs, int njobs, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {  // last job with begin <= i
      const int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].begin <= i) lo = mid; else hi = mid - 1;
    }
    const vm_pack_job& jb = jobs[lo];
    const PackGeom g = jb.flip ? pack_geom(jb.cout, jb.cin) : pack_geom(jb.cin, jb.cout);
    static_cast<bf16*>(jb.packed)[i - jb.begin] =
        __float2bfloat16_rn(pack_value(g, i - jb.begin, jb.w, jb.cin, jb.cout, jb.flip));
  }
}

extern "C" int vm_pack_weights_batch(const vm_pack_job* jobs, int njobs, int64_t total_elems, void* stream) {
  VM_REQUIRE(jobs && njobs > 0 && total_elems > 0, VM_E_ARG, "vm_pack_weights_batch: bad argument");
  k_pack_batch<<<grid_for(total_elems, 256), 256, 0, as_stream(stream)>>>(jobs, njobs, total_elems);
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

extern "C" void vm_debug_set_fwd_probe(long long* buf) { g_fwd_dbg = buf; }

extern "C" int vm_conv3d_fwd_tc(const void* x, int64_t x_bstride, const void* wpacked,
                                const float* bias, void* y, int64_t y_bstride, const void* mask,
                                int64_t mask_bstride, int B, int Cin, int Cout, int D, int H, int W,
                                unsigned flags, void* stream) {
  VM_REQUIRE(x && wpacked && y, VM_E_ARG, "vm_conv3d_fwd_tc: null pointer");
  VM_REQUIRE((flags & VM_CONV_NOBIAS) || bias, VM_E_ARG, "vm_conv3d_fwd_tc: bias required");
  VM_REQUIRE(!(flags & VM_CONV_MASK) || mask, VM_E_ARG, "vm_conv3d_fwd_tc: mask required");
  VM_REQUIRE(B > 0 && Cin > 0 && Cout > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE,
             "vm_conv3d_fwd_tc: bad shape");
  PackGeom pg = pack_geom(Cin, Cout);
  FwdParams p{};
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
  const int64_t rows = (int64_t)(D + 2) * p.P;
  p.plane8 = rows * 8;
  p.y_bstride = y_bstride ? y_bstride : default_bstride(Cout, D, H, W, 1);
  p.m_bstride = mask_bstride ? mask_bstride : default_bstride(Cout, D, H, W, 1);
  p.CG = pg.CG;
  p.KC = pg.KC;
  p.Cout = Cout;
  p.Nc = pg.Nc;
  p.nchunk = pg.nchunk;
  p.flags = flags;
  p.dbg = g_fwd_dbg;
  p.wp_magic = (uint32_t)(0x100000000ULL / (uint64_t)(W + 2)) + 1;
  p.hp_magic = (uint32_t)(0x100000000ULL / (uint64_t)(H + 2)) + 1;
  VM_REQUIRE(Cout <= 1024, VM_E_UNSUPPORTED, "vm_conv3d_fwd_tc: Cout %d > 1024", Cout);
  p.b_bytes = 9 * 2 * p.Nc * 16;
  const bool fold = pg.fold;  // packed layout and kernel are both chosen by shape
  p.TS = fold ? 126 : 128;
  const int N = fold ? 3 * p.Nc : p.Nc;  // accumulator columns per tile
  const int tiles = (int)((p.anchors + p.TS - 1) / p.TS);
  // accumulators: 2 buffers x MB x N fp32 columns <= 512
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  int MB = 256 / N;
  if (MB > 8) MB = 8;
  const int mb_fill = (int)((int64_t)tiles * B * p.nchunk / nsm);  // keep >= 1 unit per SM
  if (MB > mb_fill) MB = mb_fill;
  if (MB < 1) MB = 1;
  for (;;) {
    p.R = (MB - 1) * p.TS + 128 + 2 * p.Wp + 2;
    p.Ralloc = (p.R + 7) / 8 * 8;
    p.a_bytes = (uint32_t)p.Ralloc * 16;
    p.stage_bytes = 2 * p.a_bytes + p.b_bytes;
    p.stages = (fold ? kSmemBudget - 12 * 1024 : kSmemBudget) / (int)p.stage_bytes;  // fold: 11 KB static smem
    if (p.stages > kMaxStages) p.stages = kMaxStages;
    if (p.stages >= 2 || MB == 1) break;
    MB /= 2;
  }
  VM_REQUIRE(p.stages >= 2, VM_E_UNSUPPORTED, "vm_conv3d_fwd_tc: W=%d too wide for the stage budget", W);
  p.MB = MB;
  p.mblocks = (tiles + MB - 1) / MB;
  p.units = B * p.mblocks * p.nchunk;
  p.idesc = make_idesc_bf16(128, N, false, false);
  p.x = static_cast<const bf16*>(x);
  p.x_bstride = x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1);
  VM_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (p.x_bstride & 7) == 0, VM_E_ALIGN,
             "vm_conv3d_fwd_tc: slab must be 16-byte aligned");
  (void)rows;
  const size_t smem = (size_t)p.stages * p.stage_bytes;
  int grid = p.units < nsm ? p.units : nsm;
  if (fold) {
    cudaFuncSetAttribute(k_conv_fwd_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_conv_fwd_fold<<<grid, 320, smem, as_stream(stream)>>>(p);
  } else {
    cudaFuncSetAttribute(k_conv_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_conv_fwd_tc<<<grid, 320, smem, as_stream(stream)>>>(p);
  }
  return launch_status("vm_conv3d_fwd_tc");
}


namespace {
struct WgPlan {
  WgParams p;
  size_t ws_main, ws_bias;
};

int g_force_runs = -1, g_force_ks = 0, g_force_mpu = 0, g_force_fold = 0;  // fold: opt-in (staging-bound, see DESIGN)

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
  p.CGo = (Cout + 7) / 8;
  p.Cout = Cout;
  p.Nc = (Cout + 15) / 16 * 16;
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
  // kw folded into N (three shifted gy copies, N = 3*Nc) whenever it fits an MMA
  const int fold = (p.gwide && 3 * p.Nc <= 256 && g_force_fold > 0) ? 1 : 0;
  auto g_region = [&](int KS) -> uint32_t {  // gy bytes per stage (raw box [+ shifted copies])
    if (fold) {
      const uint32_t raw = ((uint32_t)p.CGo * (KS + 16) * 16 + 1023) & ~1023u;
      return raw + 3u * (uint32_t)(p.Nc / 8) * KS * 16;
    }
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
    return !((g_force_runs >= 0 && runs != g_force_runs) || (g_force_ks && KS != g_force_ks) ||
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
  p.fold = fold;
  p.RR = p.KS + 8;
  p.RRg = p.KS + 16;
  p.runs_alloc = (16 * p.mt_per_unit + 2) / 3 + 2;
  // TMA tensor destinations (the gy box) must be 128-byte aligned: keep every region 1 KB aligned
  p.a_bytes = ((p.runs ? (uint32_t)p.runs_alloc * 3 * p.Wp * 16 : (uint32_t)p.mt_per_unit * 16 * p.RR * 16) + 1023) & ~1023u;
  p.g_bytes = (uint32_t)p.CGo * (fold ? p.RRg : p.RR) * 16;
  p.gc_off = fold ? (((uint32_t)p.CGo * p.RRg * 16 + 1023) & ~1023u) : 0;
  p.stage_bytes = (p.a_bytes + g_region(p.KS) + 1023) & ~1023u;
  p.stages = kSmemBudget / (int)p.stage_bytes;
  if (p.stages > kMaxStages) p.stages = kMaxStages;
  VM_REQUIRE(p.stages >= 2 && p.mt_per_unit >= 1, VM_E_UNSUPPORTED, "vm_conv3d_wgrad_tc: stage does not fit");
  p.n_mtgroups = (p.MT + p.mt_per_unit - 1) / p.mt_per_unit;
  const int64_t anchors = (int64_t)D * p.P + 2;  // + kw shift of the folded B operand
  p.stages_total = (int)((anchors + p.KS - 1) / p.KS);
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  int want = (2 * nsm + p.n_mtgroups * B - 1) / (p.n_mtgroups * B);  // ~2 units per SM
  if (want < 1) want = 1;
  p.spk = (p.stages_total + want - 1) / want;
  if (p.spk < 4) p.spk = 4;
  p.ksplit = (p.stages_total + p.spk - 1) / p.spk;
  p.units = p.n_mtgroups * B * p.ksplit;
  p.idesc = make_idesc_bf16(128, p.fold ? 3 * p.Nc : p.Nc, true, true);
  p.grid = p.units;
  if (p.grid > nsm) p.grid = (nsm / p.n_mtgroups) * p.n_mtgroups;  // CTA keeps one M-tile group
  if (p.grid < p.n_mtgroups) p.grid = p.n_mtgroups;
  pl.ws_main = (size_t)(p.grid / p.n_mtgroups) * p.MT * 3 * p.Nc * 128 * sizeof(float);
  pl.ws_bias = p.ones_slot >= 0 ? 0 : bias_grad_ws_bytes((int64_t)B * D * H * W, Cout);
  return VM_OK;
}

// 4-D gy map with 128-byte inner boxes: (64 = 8 rows x 8 ch, rows/8, CG, B)
int make_wide_map(CUtensorMap* m, const void* base, int64_t bstride, int CG, int64_t rows, int B,
                  int box_blocks, int box_groups) {
  auto enc = encode_fn();
  VM_REQUIRE(enc, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  VM_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, VM_E_ALIGN, "slab base not 16B aligned");
  cuuint64_t dims[4] = {64, (cuuint64_t)(rows / 8), (cuuint64_t)CG, (cuuint64_t)B};
  cuuint64_t strides[3] = {128, (cuuint64_t)rows * 16, (cuuint64_t)bstride * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_blocks, (cuuint32_t)box_groups, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  VM_REQUIRE(r == CUDA_SUCCESS, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled (wide) failed (%d)", (int)r);
  return VM_OK;
}

int make_group_map(CUtensorMap* m, const void* base, int64_t bstride, int CG, int64_t rows, int B,
                   int box_rows, int box_groups) {
  auto enc = encode_fn();
  VM_REQUIRE(enc, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {8, (cuuint64_t)rows, (cuuint64_t)CG, (cuuint64_t)B};
  cuuint64_t strides[3] = {16, (cuuint64_t)rows * 16, (cuuint64_t)bstride * 2};
  cuuint32_t box[4] = {8, (cuuint32_t)box_rows, (cuuint32_t)box_groups, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  VM_REQUIRE(r == CUDA_SUCCESS, VM_E_UNSUPPORTED, "cuTensorMapEncodeTiled (group) failed (%d)", (int)r);
  return VM_OK;
}
}  // namespace

extern "C" void vm_debug_force_wgrad_fold(int fold) { g_force_fold = fold; }

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

extern "C" size_t vm_conv3d_wgrad_tc_ws(int B, int Cin, int Cout, int D, int H, int W) {
  WgPlan pl;
  if (plan_wgrad(B, Cin, Cout, D, H, W, pl) != VM_OK) return 0;
  return pl.ws_main + pl.ws_bias + 256;
}

extern "C" int vm_conv3d_wgrad_tc(const void* x, int64_t x_bstride, const void* gy,
                                  int64_t gy_bstride, float* gw, float* gb, void* ws, int B, int Cin,
                                  int Cout, int D, int H, int W, void* stream) {
  VM_REQUIRE(x && gy && gw && gb && ws, VM_E_ARG, "vm_conv3d_wgrad_tc: null pointer");
  VM_REQUIRE(B > 0 && Cin > 0 && Cout > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE,
             "vm_conv3d_wgrad_tc: bad shape");
  WgPlan pl;
  int rc = plan_wgrad(B, Cin, Cout, D, H, W, pl);
  if (rc) return rc;
  WgParams p = pl.p;
  p.x = static_cast<const bf16*>(x);
  p.x_bstride = x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1);
  p.ws = static_cast<float*>(ws);
  const int64_t gbs = gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1);
  const int64_t rows = (int64_t)(D + 2) * p.P;
  CUtensorMap gmap;
  rc = p.gwide ? make_wide_map(&gmap, gy, gbs, p.CGo, rows, B, (p.fold ? p.RRg : p.RR) / 8, p.CGo)
               : make_group_map(&gmap, gy, gbs, p.CGo, rows, B, p.RR, p.CGo);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  cudaFuncSetAttribute(k_conv_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
  k_conv_wgrad_tc<<<p.grid, 192, (size_t)p.stages * p.stage_bytes, st>>>(gmap, p);
  rc = launch_status("vm_conv3d_wgrad_tc");
  if (rc) return rc;
  const int nk = p.grid / p.n_mtgroups;
  const int64_t E = (int64_t)p.MT * 3 * p.Nc * 128;
  k_wgrad_tc_finalize<<<grid_for(E, 256), 256, 0, st>>>(p.ws, gw, gb, nk, p.MT, p.Nc, p.CG, Cin, Cout,
                                                         p.ones_slot, p.runs);
  rc = launch_status("vm_conv3d_wgrad_tc finalize");
  if (rc || p.ones_slot >= 0) return rc;
  float* wsb = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ((pl.ws_main + 255) / 256) * 256);
  return bias_grad_bf16(gy, gbs, gb, wsb, B, Cout, D, H, W, st);
}
