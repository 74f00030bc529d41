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
};

static PackGeom pack_geom(int cin, int cout) {
  PackGeom g;
  g.cin = cin;
  g.cout = cout;
  g.CG = (cin + 7) / 8;
  g.KC = (g.CG + 1) / 2;
  int npad = (cout + 15) / 16 * 16;
  g.nchunk = (npad + 255) / 256;
  g.Nc = ((npad + g.nchunk - 1) / g.nchunk + 15) / 16 * 16;
  return g;
}

__global__ void k_pack_weights(const float* __restrict__ w, bf16* __restrict__ out, PackGeom g,
                               int layer_cin, int layer_cout, int flip) {
  const int64_t per_tap = 2LL * g.Nc * 8;
  const int64_t total = (int64_t)g.nchunk * g.KC * 27 * per_tap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int e = i % 8;
    int64_t r = i / 8;
    int n = r % g.Nc;
    r /= g.Nc;
    int half = r % 2;
    r /= 2;
    int j = r % 9;
    r /= 9;
    int kd = r % 3;
    r /= 3;
    int kc = r % g.KC;
    int nch = (int)(r / g.KC);
    int t = kd * 9 + j;
    int ci = (kc * 2 + half) * 8 + e;
    int co = nch * g.Nc + n;
    float v = 0.f;
    if (ci < g.cin && co < g.cout) {
      if (!flip)
        v = w[((int64_t)t * layer_cin + ci) * layer_cout + co];
      else  // conv cin = layer cout, conv cout = layer cin
        v = w[((int64_t)(26 - t) * layer_cin + co) * layer_cout + ci];
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------ forward kernel
struct FwdParams {
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
};

__global__ void __launch_bounds__(192, 1)
    k_conv_fwd_tc(const __grid_constant__ CUtensorMap xmap, const FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
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
      mbar_init(&tempty[b], 128);
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
      tma_prefetch(&xmap);
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
            mbar_arrive_expect_tx(&full[stage], ng * p.a_bytes + p.b_bytes);
            for (int g = 0; g < ng; ++g)
              for (int rb = 0; rb < p.Ralloc; rb += kBoxR)
                tma_load_4d(sA + (size_t)g * p.a_bytes + (size_t)rb * 16, &xmap, &full[stage], 0,
                            (int)(a0 + (int64_t)kd * p.P + rb), kc * 2 + g, b);
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
    int stage = 0;
    uint32_t phase = 0;
    int ab = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      mbar_wait(&tempty[ab], aphase ^ 1);
      tc_fence_after();
      for (int s = 0; s < nstage_k; ++s) {
        const int kc = s / 3;
        const int ng = (kc * 2 + 1 < p.CG) ? 2 : 1;
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sB = sA + 2 * p.a_bytes;
          const uint32_t lbo_a = ng == 2 ? p.a_bytes : 0;
#pragma unroll 1
          for (int j = 0; j < 9; ++j) {
            const uint64_t bdesc = make_sdesc(sB + j * (2 * p.Nc * 16), p.Nc * 16, 128);
            const int roff = (j / 3) * p.Wp + (j % 3);
#pragma unroll 1
            for (int i = 0; i < p.MB; ++i) {
              const uint64_t adesc = make_sdesc(sA + (uint32_t)(i * 128 + roff) * 16, lbo_a, 128);
              mma_bf16_ss(tbase + (uint32_t)((ab * p.MB + i) * p.Nc), adesc, bdesc, p.idesc,
                          (s > 0 || j > 0) ? 1u : 0u);
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
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int ab = 0;
    uint32_t aphase = 0;
    const int ngroups = min(p.Nc, p.Cout) / 8;  // channel groups stored per chunk (upper bound)
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int nch = u % p.nchunk;
      const int mb = (u / p.nchunk) % p.mblocks;
      const int b = u / (p.nchunk * p.mblocks);
      const int64_t a0 = (int64_t)mb * p.MB * 128;
      mbar_wait(&tfull[ab], aphase);
      tc_fence_after();
      for (int i = 0; i < p.MB; ++i) {
        const int64_t a = a0 + i * 128 + q * 32 + lane;
        const int wq = (int)(a % p.Wp);
        const int hq = (int)((a / p.Wp) % p.Hp);
        const bool valid = a < p.anchors && wq < p.W && hq < p.H;
        const int64_t orow = a + p.P + p.Wp + 1;
        for (int g = 0; g * 8 < p.Nc; ++g) {
          uint32_t r[8];
          tmem_ld8(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * p.MB + i) * p.Nc + g * 8), r);
          tmem_ld_wait();
          const int co0 = nch * p.Nc + g * 8;
          if (valid && co0 < p.Cout) {
            float v[8];
  #pragma unroll
            for (int e = 0; e < 8; ++e) {
              v[e] = __uint_as_float(r[e]);
              if (!(p.flags & VM_CONV_NOBIAS) && co0 + e < p.Cout) v[e] += p.bias[co0 + e];
            }
            if (p.flags & VM_CONV_RELU) {
  #pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
            }
            const int cg = co0 / 8;
            if (p.flags & VM_CONV_MASK) {
              int4 mraw = *reinterpret_cast<const int4*>(p.mask + b * p.m_bstride + cg * p.plane8 + orow * 8);
              const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&mraw);
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
            *reinterpret_cast<int4*>(p.y + b * p.y_bstride + cg * p.plane8 + orow * 8) = out;
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
    (void)ngroups;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ weight-gradient kernel
// Rows of M: 16 channel groups per M-tile, group g = p*CG + cg with p = kd*3 + kh.
// Each group is staged as its own run of KS+8 rows (the (kd,kh)-shifted input),
// so consecutive groups sit at a uniform stride (SBO) and the kw shift is a
// 16-byte start-address offset along K.  B = gy rows (MN-major, co groups).
constexpr int kWgKS = 64;       // anchors per stage (K of one stage)
constexpr int kWgRows = kWgKS + 8;

struct WgParams {
  const bf16* x;
  int64_t x_bstride;
  int64_t plane8;   // elements per channel-group plane
  int B, D, H, W, Hp, Wp, P;
  int CG, CGo, Cout, Nc;
  int MT, mt_per_unit, n_mtgroups;
  int spk;          // stages per unit (K-split chunk)
  int ksplit;       // K-split chunks per sample
  int stages_total; // per sample
  int units;
  int stages;       // pipeline depth
  uint32_t a_bytes; // per stage: mt_per_unit*16 groups * kWgRows * 16
  uint32_t g_bytes; // per stage loaded: CGo * kWgKS * 16 (allocated: Nc/8 groups)
  uint32_t stage_bytes;
  uint32_t idesc;
  float* ws;        // [kidx = b*ksplit + ks][MT][3][Nc][128]
};

__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad_tc(const __grid_constant__ CUtensorMap gmap, const WgParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull, tempty;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
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
  const int ngroups_total = 9 * p.CG;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&gmap);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int mg = u % p.n_mtgroups;
        const int ks = (u / p.n_mtgroups) % p.ksplit;
        const int b = u / (p.n_mtgroups * p.ksplit);
        const int mt0 = mg * p.mt_per_unit;
        const int nmt = min(p.mt_per_unit, p.MT - mt0);
        const int s0 = ks * p.spk, s1 = min(p.stages_total, s0 + p.spk);
        for (int s = s0; s < s1; ++s) {
          const int64_t k0 = (int64_t)s * kWgKS;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + (size_t)stage * p.stage_bytes;
          uint8_t* sG = sA + p.a_bytes;
          int nvalid = 0;
          for (int i = 0; i < nmt * 16; ++i)
            if ((mt0 * 16 + i) < ngroups_total) ++nvalid;
          mbar_arrive_expect_tx(&full[stage], (uint32_t)nvalid * kWgRows * 16 + p.g_bytes);
          for (int i = 0; i < nmt * 16; ++i) {
            const int g = mt0 * 16 + i;
            if (g >= ngroups_total) break;
            const int pp = g / p.CG, cg = g % p.CG;
            const int kd = pp / 3, kh = pp % 3;
            const bf16* src = p.x + b * p.x_bstride + cg * p.plane8 + (k0 + (int64_t)kd * p.P + (int64_t)kh * p.Wp) * 8;
            bulk_load(sA + (size_t)i * kWgRows * 16, src, kWgRows * 16, &full[stage]);
          }
          for (int cgo = 0; cgo < p.CGo; ++cgo)
            tma_load_4d(sG + (size_t)cgo * kWgKS * 16, &gmap, &full[stage], 0,
                        (int)(k0 + p.P + p.Wp + 1), cgo, b);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0, tph = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int mg = u % p.n_mtgroups;
      const int ks = (u / p.n_mtgroups) % p.ksplit;
      const int mt0 = mg * p.mt_per_unit;
      const int nmt = min(p.mt_per_unit, p.MT - mt0);
      const int s0 = ks * p.spk, s1 = min(p.stages_total, s0 + p.spk);
      mbar_wait(&tempty, tph ^ 1);
      tc_fence_after();
      for (int s = s0; s < s1; ++s) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
          const uint32_t sG = sA + p.a_bytes;
#pragma unroll 1
          for (int kk = 0; kk < kWgKS / 16; ++kk) {
            const uint64_t bdesc = make_sdesc(sG + kk * 256, 128, kWgKS * 16);
#pragma unroll 1
            for (int m = 0; m < nmt; ++m)
#pragma unroll 1
              for (int kw = 0; kw < 3; ++kw) {
                const uint32_t a_addr = sA + (uint32_t)((m * 16) * kWgRows + kk * 16 + kw) * 16;
                const uint64_t adesc = make_sdesc(a_addr, 128, kWgRows * 16);
                mma_bf16_ss(tbase + (uint32_t)((m * 3 + kw) * p.Nc), adesc, bdesc, p.idesc,
                            (s > s0 || kk > 0) ? 1u : 0u);
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
      if (elect_one()) mma_commit(&tfull);
      __syncwarp();
      tph ^= 1;
    }
  } else {
    const int q = warp & 3;
    uint32_t tph = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int mg = u % p.n_mtgroups;
      const int ks = (u / p.n_mtgroups) % p.ksplit;
      const int b = u / (p.n_mtgroups * p.ksplit);
      const int mt0 = mg * p.mt_per_unit;
      const int nmt = min(p.mt_per_unit, p.MT - mt0);
      const int kidx = b * p.ksplit + ks;
      mbar_wait(&tfull, tph);
      tc_fence_after();
      const int m_row = q * 32 + lane;
      for (int m = 0; m < nmt; ++m)
        for (int kw = 0; kw < 3; ++kw)
          for (int n0 = 0; n0 < p.Nc; n0 += 8) {
            uint32_t r[8];
            tmem_ld8(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)((m * 3 + kw) * p.Nc + n0), r);
            tmem_ld_wait();
            float* dst = p.ws + ((((int64_t)kidx * p.MT + mt0 + m) * 3 + kw) * p.Nc + n0) * 128 + m_row;
#pragma unroll
            for (int e = 0; e < 8; ++e) dst[e * 128] = __uint_as_float(r[e]);
          }
      tc_fence_before();
      mbar_arrive(&tempty);
      tph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// gw[t][ci][co] = sum_k ws[k][mt][kw][co][m], t = (kd*3+kh)*3 + kw, g = (kd*3+kh)*CG + ci/8
__global__ void k_wgrad_tc_finalize(const float* __restrict__ ws, float* __restrict__ gw, int nk, int MT,
                                    int Nc, int CG, int Cin, int Cout) {
  const int64_t n = (int64_t)27 * Cin * Cout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int co = i % Cout;
    const int ci = (i / Cout) % Cin;
    const int t = (int)(i / ((int64_t)Cout * Cin));
    const int pp = t / 3, kw = t % 3;
    const int g = pp * CG + ci / 8;
    const int mt = g / 16, m = (g % 16) * 8 + (ci % 8);
    float s = 0.f;
    for (int k = 0; k < nk; ++k) s += ws[((((int64_t)k * MT + mt) * 3 + kw) * Nc + co) * 128 + m];
    gw[i] = s;
  }
}

}  // namespace vm

using namespace vm;

extern "C" size_t vm_packed_weights_bytes(int Cin, int Cout) {
  PackGeom g = pack_geom(Cin, Cout);
  return (size_t)g.nchunk * g.KC * 27 * 2 * g.Nc * 8 * sizeof(bf16);
}

extern "C" int vm_pack_weights(const float* w, void* packed, int Cin, int Cout, int flip, void* stream) {
  VM_REQUIRE(w && packed && Cin > 0 && Cout > 0, VM_E_ARG, "vm_pack_weights: bad argument");
  PackGeom g = flip ? pack_geom(Cout, Cin) : pack_geom(Cin, Cout);
  int64_t total = (int64_t)vm_packed_weights_bytes(g.cin, g.cout) / 2;
  k_pack_weights<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(w, (bf16*)packed, g, Cin, Cout, flip);
  return launch_status("vm_pack_weights");
}

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
  p.b_bytes = 9 * 2 * p.Nc * 16;
  const int tiles = (int)((p.anchors + 127) / 128);
  // accumulators: 2 buffers x MB x Nc fp32 columns <= 512
  int MB = 256 / p.Nc;
  if (MB > 8) MB = 8;
  if (MB > tiles) MB = tiles;
  if (MB < 1) MB = 1;
  for (;;) {
    const int R = MB * 128 + 2 * p.Wp + 2;
    p.Ralloc = (R + kBoxR - 1) / kBoxR * kBoxR;
    p.a_bytes = (uint32_t)p.Ralloc * 16;
    p.stage_bytes = 2 * p.a_bytes + p.b_bytes;
    p.stages = kSmemBudget / (int)p.stage_bytes;
    if (p.stages > kMaxStages) p.stages = kMaxStages;
    if (p.stages >= 2 || MB == 1) break;
    MB /= 2;
  }
  VM_REQUIRE(p.stages >= 2, VM_E_UNSUPPORTED, "vm_conv3d_fwd_tc: W=%d too wide for the stage budget", W);
  p.MB = MB;
  p.mblocks = (tiles + MB - 1) / MB;
  p.units = B * p.mblocks * p.nchunk;
  p.idesc = make_idesc_bf16(128, p.Nc, false, false);
  CUtensorMap xmap;
  int64_t xb = x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1);
  int rc = make_slab_map(&xmap, x, xb, p.CG, rows, B, kBoxR);
  if (rc) return rc;
  const size_t smem = (size_t)p.stages * p.stage_bytes;
  cudaFuncSetAttribute(k_conv_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
  int nsm = vm_num_sms(0);
  int grid = p.units < nsm ? p.units : nsm;
  k_conv_fwd_tc<<<grid, 192, smem, as_stream(stream)>>>(xmap, p);
  return launch_status("vm_conv3d_fwd_tc");
}


namespace {
struct WgPlan {
  WgParams p;
  size_t ws_main, ws_bias;
};

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
  p.plane8 = (int64_t)(D + 2) * p.P * 8;
  p.CG = (Cin + 7) / 8;
  p.CGo = (Cout + 7) / 8;
  p.Cout = Cout;
  p.Nc = (Cout + 15) / 16 * 16;
  VM_REQUIRE(3 * p.Nc <= 512, VM_E_UNSUPPORTED, "vm_conv3d_wgrad_tc: Cout %d > 160 not supported yet", Cout);
  p.MT = (9 * p.CG + 15) / 16;
  p.mt_per_unit = 512 / (3 * p.Nc);
  if (p.mt_per_unit > p.MT) p.mt_per_unit = p.MT;
  // stage smem must allow >= 2 stages
  for (;;) {
    p.a_bytes = (uint32_t)p.mt_per_unit * 16 * kWgRows * 16;
    p.g_bytes = (uint32_t)p.CGo * kWgKS * 16;
    p.stage_bytes = p.a_bytes + (uint32_t)(p.Nc / 8) * kWgKS * 16;
    p.stages = kSmemBudget / (int)p.stage_bytes;
    if (p.stages >= 2 || p.mt_per_unit == 1) break;
    p.mt_per_unit--;
  }
  if (p.stages > kMaxStages) p.stages = kMaxStages;
  VM_REQUIRE(p.stages >= 2, VM_E_UNSUPPORTED, "vm_conv3d_wgrad_tc: stage does not fit");
  p.n_mtgroups = (p.MT + p.mt_per_unit - 1) / p.mt_per_unit;
  const int64_t anchors = (int64_t)D * p.P;
  p.stages_total = (int)((anchors + kWgKS - 1) / kWgKS);
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  int want = (2 * nsm + p.n_mtgroups * B - 1) / (p.n_mtgroups * B);  // ~2 units per SM
  if (want < 1) want = 1;
  p.spk = (p.stages_total + want - 1) / want;
  if (p.spk < 4) p.spk = 4;
  p.ksplit = (p.stages_total + p.spk - 1) / p.spk;
  p.units = p.n_mtgroups * B * p.ksplit;
  p.idesc = make_idesc_bf16(128, p.Nc, true, true);
  pl.ws_main = (size_t)B * p.ksplit * p.MT * 3 * p.Nc * 128 * sizeof(float);
  pl.ws_bias = bias_grad_ws_bytes((int64_t)B * D * H * W, Cout);
  return VM_OK;
}
}  // namespace

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
  rc = make_slab_map(&gmap, gy, gbs, p.CGo, rows, B, kWgKS);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  cudaFuncSetAttribute(k_conv_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
  int nsm = vm_num_sms(0);
  int grid = p.units < nsm ? p.units : nsm;
  k_conv_wgrad_tc<<<grid, 192, (size_t)p.stages * p.stage_bytes, st>>>(gmap, p);
  rc = launch_status("vm_conv3d_wgrad_tc");
  if (rc) return rc;
  const int nk = B * p.ksplit;
  k_wgrad_tc_finalize<<<grid_for((int64_t)27 * Cin * Cout, 256), 256, 0, st>>>(p.ws, gw, nk, p.MT, p.Nc, p.CG,
                                                                               Cin, Cout);
  rc = launch_status("vm_conv3d_wgrad_tc finalize");
  if (rc) return rc;
  float* wsb = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ((pl.ws_main + 255) / 256) * 256);
  return bias_grad_bf16(gy, gbs, gb, wsb, B, Cout, D, H, W, st);
}
