// first_layer.cu — the Cin = 1 convolution (the U-Net's first conv, `unet.py:191-225` enc0
// conv0 on the single-channel CT volume) forward and weight gradient as im2col tcgen05 GEMMs.
//
// With one input channel the channel-blocked kernels waste 7/8 of every K step (the input
// slab carries 8 channels, 7 of them zero) and issue as many MMAs as a 16-channel layer.
// Here the 27 taps are the K dimension instead: each thread builds one anchor row of an
// im2col tile in shared memory (27 taps + 1 ones column + 4 zeros = 32 bf16), and
//   forward:  y[a][co]  = relu(b[co] + sum_t A[a][t] W[t][co])      M = 128 anchors, N = Cout, K = 32
//   wgrad:    dW[t][co] = sum_a A[a][t] gy[a + P + Wp + 1][co]      M = 64 taps, N = Cout, K = anchors
// The same tile is the K-major A of the forward and the MN-major A of the weight gradient
// (8 taps x 8 anchors core matrices, 16 B rows).  Column 27 of A is 1 in the weight gradient,
// so row 27 of dW is the bias gradient (gy is zero on margin rows).  Reference: ops.py:69-97
// (forward), ops.py:117-138 (parameter gradients).
#include "sm100.cuh"
#include "vm_common.cuh"

namespace vm {
namespace {

using bf16 = __nv_bfloat16;

struct C1Params {
  const bf16* x;  // compact padded input [B][(D+2)(H+2)(W+2)] (vm_dense_to_compact1), zero margins
  int64_t x_bstride;
  const float* w;  // [27][Cout] fp32 (reference layout with Cin = 1)
  const float* bias;
  bf16* y;
  int64_t y_bstride;
  const bf16* gy;
  int64_t gy_bstride;
  float* ws;  // weight gradient partials [gridDim][32 taps][Nc]
  int B, D, H, W, Hp, Wp, P;
  int64_t anchors;  // D*P per sample
  int64_t plane8;   // (D+2)*P*8 elements per channel-group plane
  int Cout, Nc, tiles_per_sample, tiles;
  unsigned flags;
  uint32_t wp_magic, hp_magic, tps_magic;
};

// x / d for the small divisors of this file (multiply-high by floor(2^32 / d) + 1, corrected)
__device__ __forceinline__ uint32_t c1_div(uint32_t x, uint32_t d, uint32_t magic) {
  uint32_t q = __umulhi(x, magic);
  if (q * d > x) --q;
  if ((q + 1) * d <= x) ++q;
  return q;
}

constexpr int kC1Threads = 128;
constexpr uint32_t kC1TileBytes = 128 * 16;  // one 8-tap column group of the 128-row tile

// Row `row` of the im2col tile for anchor a: A[kg][row][8 taps], tap t = kd*9 + kh*3 + kw
// reads input row a + kd*P + kh*Wp + kw; t = 27 is the ones column (weight gradient only).
// Gathered into registers first (c1_gather) so that the next tile's loads overlap the current
// tile's MMA and drain, then stored (c1_store).
__device__ __forceinline__ void c1_gather(const C1Params& p, const bf16* xb, int64_t a, bool in, bool ones,
                                          uint32_t (&v)[16]) {
  // 9 (kd, kh) row offsets in 32-bit element units (a sample is < 2^31 elements, c1_setup);
  // the 3 kw taps of a row are immediate offsets of one address (the per-tap index arithmetic
  // made the forward instruction-issue bound: ncu, issue slots 67% active)
  const uint16_t* xs = reinterpret_cast<const uint16_t*>(xb);
  const uint32_t a32 = (uint32_t)a;
  uint32_t h[28];
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    const uint16_t* rp = xs + (a32 + (uint32_t)((r / 3) * p.P + (r % 3) * p.Wp));
#pragma unroll
    for (int kw = 0; kw < 3; ++kw) h[r * 3 + kw] = in ? (uint32_t)__ldg(rp + kw) : 0u;
  }
  h[27] = (ones && in) ? 0x3F80u : 0u;  // tap 27 = bf16 1.0
#pragma unroll
  for (int i = 0; i < 14; ++i) v[i] = __byte_perm(h[2 * i], h[2 * i + 1], 0x5410);
  v[14] = 0u;
  v[15] = 0u;
}
__device__ __forceinline__ void c1_store(const uint32_t (&v)[16], uint8_t* sA, int row) {
#pragma unroll
  for (int kg = 0; kg < 4; ++kg)
    *reinterpret_cast<uint4*>(sA + kg * kC1TileBytes + row * 16) =
        make_uint4(v[4 * kg], v[4 * kg + 1], v[4 * kg + 2], v[4 * kg + 3]);
}

// output row of anchor a and whether it is an interior voxel
__device__ __forceinline__ int64_t c1_anchor_row(const C1Params& p, int64_t a, bool& valid) {
  const uint32_t au = (uint32_t)a;
  uint32_t qa = __umulhi(au, p.wp_magic);
  if (qa * (uint32_t)p.Wp > au) --qa;
  if ((qa + 1) * (uint32_t)p.Wp <= au) ++qa;
  const int wq = (int)(au - qa * (uint32_t)p.Wp);
  uint32_t qh = __umulhi(qa, p.hp_magic);
  if (qh * (uint32_t)p.Hp > qa) --qh;
  if ((qh + 1) * (uint32_t)p.Hp <= qa) ++qh;
  const int hq = (int)(qa - qh * (uint32_t)p.Hp);
  valid = a < p.anchors && wq < p.W && hq < p.H;
  return a + p.P + p.Wp + 1;
}

// Forward.  One 128-anchor tile per iteration; many small CTAs per SM (9 KB shared memory,
// 32 TMEM columns) overlap one CTA's gathers with another's MMA and drain.
__global__ void __launch_bounds__(kC1Threads) k_c1_fwd(const C1Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float sbias[32];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 4 * kC1TileBytes;  // [kg][n][8 taps]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<32>(&tslot);
  pdl_wait();
  pdl_trigger();
  // weights -> bf16 K-major B tile (taps >= 27 and co >= Cout zero); bias in fp32
  for (int i = threadIdx.x; i < 4 * p.Nc * 8; i += kC1Threads) {
    const int kk = i % 8, n = (i / 8) % p.Nc, t = (i / (8 * p.Nc)) * 8 + kk;
    reinterpret_cast<bf16*>(sB)[i] = __float2bfloat16_rn(t < 27 && n < p.Cout ? p.w[t * p.Cout + n] : 0.f);
  }
  if (threadIdx.x < 32)
    sbias[threadIdx.x] = (threadIdx.x < p.Cout && !(p.flags & VM_CONV_NOBIAS)) ? p.bias[threadIdx.x] : 0.f;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t idesc = make_idesc_bf16(128, p.Nc, false, false);
  const int row = threadIdx.x;
  uint32_t phase = 0;
  uint32_t v[16];
  auto tile_anchor = [&](int tile, int& b) -> int64_t {
    b = (int)c1_div((uint32_t)tile, (uint32_t)p.tiles_per_sample, p.tps_magic);
    return (int64_t)(tile - b * p.tiles_per_sample) * 128 + row;
  };
  if ((int)blockIdx.x < p.tiles) {
    int b0;
    const int64_t a0 = tile_anchor(blockIdx.x, b0);
    c1_gather(p, p.x + b0 * p.x_bstride, a0, a0 < p.anchors, false, v);
  }
  for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    int b;
    const int64_t a = tile_anchor(tile, b);
    c1_store(v, sA, row);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint64_t ad = make_sdesc(smem_u32(sA), kC1TileBytes, 128);
      const uint64_t bd = make_sdesc(smem_u32(sB), (uint32_t)p.Nc * 16, 128);
      mma_bf16_ss(tbase, ad, bd, idesc, 0u);
      mma_bf16_ss(tbase, ad + ((2 * kC1TileBytes) >> 4), bd + ((2u * p.Nc * 16) >> 4), idesc, 1u);
      mma_commit(&mbar);
    }
    if (tile + (int)gridDim.x < p.tiles) {  // next tile's gathers overlap this tile's MMA and drain
      int bn;
      const int64_t an = tile_anchor(tile + gridDim.x, bn);
      c1_gather(p, p.x + bn * p.x_bstride, an, an < p.anchors, false, v);
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    tc_fence_after();
    bool valid;
    const int64_t orow = c1_anchor_row(p, a, valid);
    bf16* yb = p.y + b * p.y_bstride;
    for (int g = 0; g < p.Nc / 8; ++g) {
      uint32_t r[8];
      tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)(g * 8), r);
      tmem_ld_wait();
      const float4 b0 = *reinterpret_cast<const float4*>(&sbias[g * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&sbias[g * 8 + 4]);
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      int4 out;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v0 = __uint_as_float(r[2 * e]) + bb[2 * e], v1 = __uint_as_float(r[2 * e + 1]) + bb[2 * e + 1];
        if (g * 8 + 2 * e >= p.Cout) v0 = 0.f;
        if (g * 8 + 2 * e + 1 >= p.Cout) v1 = 0.f;
        ow[e] = (p.flags & VM_CONV_RELU) ? pack_bf16x2_relu(v0, v1) : pack_bf16x2(v0, v1);
      }
      if (valid) *reinterpret_cast<int4*>(yb + g * p.plane8 + orow * 8) = out;
    }
    tc_fence_before();
    __syncthreads();  // TMEM drained and the tile consumed before the next build / MMA
  }
  (void)lane;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tbase);
}

// Weight gradient: each CTA accumulates its tiles in TMEM (M = 64 taps, N = Nc) and writes
// one fp32 partial; k_c1_wgrad_finalize sums the partials in CTA order (deterministic).
__global__ void __launch_bounds__(kC1Threads) k_c1_wgrad(const C1Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  uint8_t* sA = smem;                        // [8 kg][128 rows][16 B]; kg 4..7 stay zero (M = 64)
  uint8_t* sG = smem + 8 * kC1TileBytes;     // [Nc/8][128 rows][16 B]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 4 * (int)kC1TileBytes / 16; i += kC1Threads)
    reinterpret_cast<uint4*>(sA + 4 * kC1TileBytes)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<32>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tbase = tslot;
  const uint32_t idesc = make_idesc_bf16(64, p.Nc, true, true);
  const int row = threadIdx.x;
  const int ng = p.Nc / 8;
  uint32_t phase = 0;
  bool any = false;
  uint32_t v[16];
  int4 gv[4];  // Nc <= 32: up to 4 channel groups of gy
  auto gather = [&](int tile) {
    const int b = (int)c1_div((uint32_t)tile, (uint32_t)p.tiles_per_sample, p.tps_magic);
    const int64_t a = (int64_t)(tile - b * p.tiles_per_sample) * 128 + row;
    const bool in = a < p.anchors;
    c1_gather(p, p.x + b * p.x_bstride, a, in, true, v);
    const bf16* gyb = p.gy + b * p.gy_bstride + (a + p.P + p.Wp + 1) * 8;
#pragma unroll
    for (int g = 0; g < 4; ++g)
      gv[g] = in && g < ng && g * 8 < p.Cout ? __ldg(reinterpret_cast<const int4*>(gyb + g * p.plane8))
                                             : make_int4(0, 0, 0, 0);
  };
  if ((int)blockIdx.x < p.tiles) gather(blockIdx.x);
  for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    c1_store(v, sA, row);
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (g < ng) *reinterpret_cast<int4*>(sG + g * kC1TileBytes + row * 16) = gv[g];
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint64_t ad = make_sdesc(smem_u32(sA), 128, kC1TileBytes);
      const uint64_t bd = make_sdesc(smem_u32(sG), 128, kC1TileBytes);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)  // 16 anchors (256 B) per MMA
        mma_bf16_ss(tbase, ad + (uint64_t)(kk * 16), bd + (uint64_t)(kk * 16), idesc, (any || kk > 0) ? 1u : 0u);
      mma_commit(&mbar);
    }
    any = true;
    if (tile + (int)gridDim.x < p.tiles) gather(tile + gridDim.x);  // overlaps the MMAs
    mbar_wait(&mbar, phase);  // the MMAs have read the tile before it is rebuilt
    phase ^= 1u;
    tc_fence_after();
  }
  // drain: M = 64 rows m live in TMEM lanes (m/16)*32 + m%16 — lanes 0..15 of each warp
  float* dst = p.ws + (int64_t)blockIdx.x * 32 * p.Nc;
  const int m = warp * 16 + lane;
  for (int g = 0; g < ng; ++g) {
    uint32_t r[8];
    tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)(g * 8), r);
    tmem_ld_wait();
    if (lane < 16 && m < 32) {
#pragma unroll
      for (int e = 0; e < 8; ++e) dst[m * p.Nc + g * 8 + e] = any ? __uint_as_float(r[e]) : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tbase);
}

// gw[t][co] (t < 27) and gb[co] (ones column t = 27): partials summed in CTA order
__global__ void __launch_bounds__(256) k_c1_wgrad_finalize(const float* __restrict__ ws, int nparts, int Nc,
                                                           int Cout, float* __restrict__ gw, float* __restrict__ gb) {
  pdl_wait();
  __shared__ float red[8][32];
  const int o = blockIdx.x;  // (t, co), t < 28
  const int t = o / Cout, co = o % Cout;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float s = 0.f;
  for (int k = threadIdx.x; k < nparts; k += 256) s += ws[(int64_t)k * 32 * Nc + t * Nc + co];
  // fixed-order tree: lanes, then warps
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) red[0][w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int i = 0; i < 8; ++i) tot += red[0][i];
    if (t < 27)
      gw[t * Cout + co] = tot;
    else
      gb[co] = tot;
  }
}

int c1_setup(C1Params& p, int B, int Cout, int D, int H, int W) {
  VM_REQUIRE(B > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE, "first-layer conv: bad shape");
  VM_REQUIRE(Cout > 0 && Cout <= 32, VM_E_UNSUPPORTED, "first-layer conv: Cout %d > 32", Cout);
  p.B = B;
  p.D = D;
  p.H = H;
  p.W = W;
  p.Hp = H + 2;
  p.Wp = W + 2;
  p.P = p.Hp * p.Wp;
  p.anchors = (int64_t)D * p.P;
  p.plane8 = (int64_t)(D + 2) * p.P * 8;
  p.Cout = Cout;
  p.Nc = Cout <= 16 ? 16 : 32;
  p.tiles_per_sample = (int)((p.anchors + 127) / 128);
  p.tiles = B * p.tiles_per_sample;
  p.wp_magic = fastdiv_magic((uint32_t)p.Wp);
  p.hp_magic = fastdiv_magic((uint32_t)p.Hp);
  p.tps_magic = fastdiv_magic((uint32_t)p.tiles_per_sample);
  VM_REQUIRE((int64_t)(D + 2) * p.P < (1LL << 31), VM_E_SHAPE, "first-layer conv: sample too large");
  return VM_OK;
}

constexpr int kC1WgCtasPerSm = 16;  // weight gradient: cap on the partial count (occupancy binds first)

// One wave: as many CTAs as are resident at once (a second partial wave cost 1.33x).  The
// runtime occupancy query answers 1 CTA/SM for these TMEM-allocating kernels, so the limit is
// computed from the kernel's registers and shared memory (32 TMEM columns per CTA never bind).
template <typename K>
int c1_grid(K kern, size_t smem, int tiles, int cap_per_sm) {
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  cudaFuncAttributes fa{};
  int per_sm = 1;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) {
    const int warps = kC1Threads / 32;
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / (regs_warp * warps);
    const int by_smem = (228 * 1024) / (int)(smem + fa.sharedSizeBytes + 1024);
    const int by_threads = 2048 / kC1Threads;
    per_sm = by_regs < by_smem ? by_regs : by_smem;
    if (by_threads < per_sm) per_sm = by_threads;
    if (per_sm > 16) per_sm = 16;  // 16 x 32 TMEM columns = 512
    if (per_sm < 1) per_sm = 1;
  }
  if (cap_per_sm > 0 && per_sm > cap_per_sm) per_sm = cap_per_sm;
  return tiles < nsm * per_sm ? tiles : nsm * per_sm;
}

}  // namespace
}  // namespace vm

using namespace vm;

// y = conv3d(x, w) (+ bias, ReLU) for a single input channel; w is the fp32 reference kernel
// [3][3][3][1][Cout] (packed to bf16 inside the kernel, so no repack after an SGD step).
extern "C" int vm_conv3d_fwd_c1(const void* x, int64_t x_bstride, const float* w, const float* bias, void* y,
                                int64_t y_bstride, int B, int Cout, int D, int H, int W, unsigned flags,
                                void* stream) {
  VM_REQUIRE(x && w && y, VM_E_ARG, "vm_conv3d_fwd_c1: null pointer");
  VM_REQUIRE((flags & VM_CONV_NOBIAS) || bias, VM_E_ARG, "vm_conv3d_fwd_c1: bias required");
  VM_REQUIRE(!(flags & VM_CONV_MASK), VM_E_UNSUPPORTED, "vm_conv3d_fwd_c1: no mask epilogue");
  C1Params p{};
  int rc = c1_setup(p, B, Cout, D, H, W);
  if (rc) return rc;
  p.x = static_cast<const bf16*>(x);
  p.x_bstride = x_bstride ? x_bstride : (int64_t)(D + 2) * (H + 2) * (W + 2);
  p.w = w;
  p.bias = bias;
  p.y = static_cast<bf16*>(y);
  p.y_bstride = y_bstride ? y_bstride : default_bstride(Cout, D, H, W, 1);
  p.flags = flags;
  const size_t smem = 4 * kC1TileBytes + 4 * (size_t)p.Nc * 16;
  launch_pdl(k_c1_fwd, c1_grid(k_c1_fwd, smem, p.tiles, 0), kC1Threads, smem, as_stream(stream), p);
  return launch_status("vm_conv3d_fwd_c1");
}

extern "C" size_t vm_conv3d_wgrad_c1_ws(int B, int Cout, int D, int H, int W) {
  C1Params p{};
  if (c1_setup(p, B, Cout, D, H, W)) return 0;
  const size_t smem = 8 * kC1TileBytes + (size_t)(p.Nc / 8) * kC1TileBytes;
  return (size_t)c1_grid(k_c1_wgrad, smem, p.tiles, kC1WgCtasPerSm) * 32 * p.Nc * sizeof(float) + 256;
}

// gw[27][1][Cout] and gb[Cout] for a single input channel (deterministic)
extern "C" int vm_conv3d_wgrad_c1(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride, float* gw,
                                  float* gb, void* ws, int B, int Cout, int D, int H, int W, void* stream) {
  VM_REQUIRE(x && gy && gw && gb && ws, VM_E_ARG, "vm_conv3d_wgrad_c1: null pointer");
  C1Params p{};
  int rc = c1_setup(p, B, Cout, D, H, W);
  if (rc) return rc;
  p.x = static_cast<const bf16*>(x);
  p.x_bstride = x_bstride ? x_bstride : (int64_t)(D + 2) * (H + 2) * (W + 2);
  p.gy = static_cast<const bf16*>(gy);
  p.gy_bstride = gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1);
  p.ws = static_cast<float*>(ws);
  const size_t smem = 8 * kC1TileBytes + (size_t)(p.Nc / 8) * kC1TileBytes;
  const int grid = c1_grid(k_c1_wgrad, smem, p.tiles, kC1WgCtasPerSm);
  cudaStream_t st = as_stream(stream);
  launch_pdl(k_c1_wgrad, grid, kC1Threads, smem, st, p);
  rc = launch_status("vm_conv3d_wgrad_c1");
  if (rc) return rc;
  launch_pdl(k_c1_wgrad_finalize, 28 * Cout, 256, 0, st, (const float*)p.ws, grid, p.Nc, Cout, gw, gb);
  return launch_status("vm_conv3d_wgrad_c1 finalize");
}

// resident CTAs per SM of the first-layer kernels as the launcher computes them (diagnostics)
extern "C" int vm_debug_c1_occupancy(int which, int Nc) {
  const size_t smem = which == 0 ? 4 * kC1TileBytes + 4 * (size_t)Nc * 16
                                 : 8 * kC1TileBytes + (size_t)(Nc / 8) * kC1TileBytes;
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  return (which == 0 ? c1_grid(k_c1_fwd, smem, 1 << 30, 0) : c1_grid(k_c1_wgrad, smem, 1 << 30, kC1WgCtasPerSm)) / nsm;
}
