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

extern "C" size_t vm_conv3d_wgrad_tc_ws(int B, int Cin, int Cout, int D, int H, int W) {
  return vm_conv3d_wgrad_simt_ws(B, Cin, Cout, D, H, W);
}

extern "C" int vm_conv3d_wgrad_tc(const void* x, int64_t x_bstride, const void* gy,
                                  int64_t gy_bstride, float* gw, float* gb, void* ws, int B, int Cin,
                                  int Cout, int D, int H, int W, void* stream) {
  // First version: the tensor-core weight-gradient kernel is not written yet; the
  // bf16 SIMT kernel computes the same quantity on CUDA cores.
  return vm_conv3d_wgrad_simt(VM_BF16, x, x_bstride, gy, gy_bstride, gw, gb, ws, B, Cin, Cout, D, H,
                              W, stream);
}
