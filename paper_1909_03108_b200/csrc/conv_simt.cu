// conv_simt.cu — CUDA-core (FFMA) conv3d forward / weight-gradient on slabs.
//
// This is the fp32 parity path (BASELINE cfg1: fp32, rel-L2 <= 1e-5 vs the f64
// oracle) and the on-device cross-check of the tcgen05 kernels; the bf16 train
// step uses conv_tc.cu.  Semantics (reference):
//   forward  conv3d_local            ops.py:69-97   (bias, then taps kz-ky-kx, channel contraction)
//   dgrad    conv3d_input_grad_local ops.py:100-114 == forward of the output gradient with
//            flipped, transposed taps (vm_weight_flip_transpose) on a halo-padded gradient slab
//   wgrad    conv3d_param_grads_local ops.py:117-138 (split-K over voxels, fixed-order reduce)
#include "vm_common.cuh"

namespace vm {

template <typename T> struct Vec8;
template <> struct Vec8<float> {
  __device__ __forceinline__ static void load(const float* p, float (&v)[8]) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ __forceinline__ static void store(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <> struct Vec8<__nv_bfloat16> {
  __device__ __forceinline__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    int4 raw = *reinterpret_cast<const int4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    int4 raw;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<int4*>(p) = raw;
  }
};

// One thread = one interior output voxel x 8 output channels (one channel block).
// Weights for the current input channel block are staged in shared memory.
template <typename T>
__global__ void __launch_bounds__(128) k_conv_fwd_simt(const T* __restrict__ x, Slab gx,
                                                       const float* __restrict__ w,
                                                       const float* __restrict__ bias,
                                                       T* __restrict__ y, Slab gy,
                                                       const T* __restrict__ mask, Slab gm, int B,
                                                       int Cin, int Cout, unsigned flags) {
  __shared__ float sw[27][8][8];
  const int cgo = blockIdx.y;
  const int64_t nvox = (int64_t)B * gy.D * gy.H * gy.W;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool active = v < nvox;
  int b = 0, d = 0, h = 0, wv = 0;
  if (active) {
    wv = v % gy.W;
    int64_t r = v / gy.W;
    h = r % gy.H;
    r /= gy.H;
    d = r % gy.D;
    b = (int)(r / gy.D);
  }
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int co = cgo * 8 + j;
    acc[j] = (!(flags & VM_CONV_NOBIAS) && co < Cout) ? bias[co] : 0.f;
  }
  const int cgin = (Cin + 7) / 8;
  for (int cgi = 0; cgi < cgin; ++cgi) {
    __syncthreads();
    for (int i = threadIdx.x; i < 27 * 64; i += blockDim.x) {
      int t = i / 64, ci = (i / 8) % 8, co = i % 8;
      int gci = cgi * 8 + ci, gco = cgo * 8 + co;
      sw[t][ci][co] = (gci < Cin && gco < Cout) ? w[((int64_t)t * Cin + gci) * Cout + gco] : 0.f;
    }
    __syncthreads();
    if (active) {
      const T* xb = x + b * gx.bstride + cgi * gx.plane();
#pragma unroll 1
      for (int kd = 0; kd < 3; ++kd)
#pragma unroll 1
        for (int kh = 0; kh < 3; ++kh)
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) {
            // padded coordinate of the tap: interior (d,h,w) sits at (d+m, h+m, w+m)
            int pd = d + gx.m - 1 + kd, ph = h + gx.m - 1 + kh, pw = wv + gx.m - 1 + kw;
            float xv[8];
            Vec8<T>::load(xb + (((int64_t)pd * gx.Hp() + ph) * gx.Wp() + pw) * 8, xv);
            const int t = (kd * 3 + kh) * 3 + kw;
#pragma unroll
            for (int ci = 0; ci < 8; ++ci)
#pragma unroll
              for (int co = 0; co < 8; ++co) acc[co] = fmaf(xv[ci], sw[t][ci][co], acc[co]);
          }
    }
  }
  if (!active) return;
  if (flags & VM_CONV_RELU) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fmaxf(acc[j], 0.f);
  }
  if (flags & VM_CONV_MASK) {
    float mv[8];
    Vec8<T>::load(mask + gm.at(b, cgo, d, h, wv), mv);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = mv[j] > 0.f ? acc[j] : 0.f;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (cgo * 8 + j >= Cout) acc[j] = 0.f;
  Vec8<T>::store(y + gy.at(b, cgo, d, h, wv), acc);
}

// Weight-gradient partials.  grid = (27 * CGin * CGout, nsplit); each block reduces
// its voxel chunk for one (tap, ci-block, co-block) to 64 values (fixed order).
template <typename T>
__global__ void __launch_bounds__(256) k_conv_wgrad_simt(const T* __restrict__ x, Slab gx,
                                                         const T* __restrict__ gy, Slab gg,
                                                         float* __restrict__ ws, int B, int CGin,
                                                         int CGout, int64_t chunk) {
  __shared__ float red[8][65];
  const int combo = blockIdx.x;  // x: 27*CGin*CGout exceeds grid.y's 65535 for 512 -> 512
  const int t = combo / (CGin * CGout);
  const int cgi = (combo / CGout) % CGin;
  const int cgo = combo % CGout;
  const int kd = t / 9, kh = (t / 3) % 3, kw = t % 3;
  const int64_t nvox = (int64_t)B * gg.D * gg.H * gg.W;
  const int64_t v0 = blockIdx.y * chunk;
  const int64_t v1 = min(nvox, v0 + chunk);
  float acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.f;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    int wv = v % gg.W;
    int64_t r = v / gg.W;
    int h = r % gg.H;
    r /= gg.H;
    int d = r % gg.D;
    int b = (int)(r / gg.D);
    float xv[8], gv[8];
    int pd = d + gx.m - 1 + kd, ph = h + gx.m - 1 + kh, pw = wv + gx.m - 1 + kw;
    Vec8<T>::load(x + b * gx.bstride + cgi * gx.plane() + (((int64_t)pd * gx.Hp() + ph) * gx.Wp() + pw) * 8, xv);
    Vec8<T>::load(gy + gg.at(b, cgo, d, h, wv), gv);
#pragma unroll
    for (int ci = 0; ci < 8; ++ci)
#pragma unroll
      for (int co = 0; co < 8; ++co) acc[ci * 8 + co] = fmaf(xv[ci], gv[co], acc[ci * 8 + co]);
  }
  // warp tree reduction, then fixed-order sum over the 8 warps
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    float s = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    acc[i] = s;
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 64; ++i) red[warp][i] = acc[i];
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    float s = 0.f;
    for (int wi = 0; wi < 8; ++wi) s += red[wi][threadIdx.x];
    const int ci = threadIdx.x / 8, co = threadIdx.x % 8;
    // ws layout: [split][t][CGin*8][CGout*8]
    int64_t idx = (((int64_t)blockIdx.y * 27 + t) * (CGin * 8) + cgi * 8 + ci) * (CGout * 8) + cgo * 8 + co;
    ws[idx] = s;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_bias_grad_partial(const T* __restrict__ gy, Slab gg,
                                                           float* __restrict__ ws, int B, int CGout,
                                                           int64_t chunk) {
  pdl_wait();
  __shared__ float red[8][9];
  const int cgo = blockIdx.y;
  const int64_t nvox = (int64_t)B * gg.D * gg.H * gg.W;
  const int64_t v0 = blockIdx.x * chunk, v1 = min(nvox, v0 + chunk);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    // 32-bit multiply-high split (nvox < 2^31, checked by the launchers; the 64-bit divisions
    // made this 1 MB reduction take ~8 us at 16^3 x 128 channels)
    const uint32_t v32 = (uint32_t)v;
    const uint32_t q1 = fastdiv(v32, (uint32_t)gg.W, gg.mW);
    const int wv = (int)(v32 - q1 * (uint32_t)gg.W);
    const uint32_t q2 = fastdiv(q1, (uint32_t)gg.H, gg.mH);
    const int h = (int)(q1 - q2 * (uint32_t)gg.H);
    const uint32_t q3 = fastdiv(q2, (uint32_t)gg.D, gg.mD);
    const int d = (int)(q2 - q3 * (uint32_t)gg.D);
    const int b = (int)q3;
    float gv[8];
    Vec8<T>::load(gy + gg.at(b, cgo, d, h, wv), gv);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += gv[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float s = acc[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    acc[j] = s;
  }
  if (threadIdx.x % 32 == 0)
    for (int j = 0; j < 8; ++j) red[threadIdx.x / 32][j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 8) {
    float s = 0.f;
    for (int wi = 0; wi < 8; ++wi) s += red[wi][threadIdx.x];
    ws[(int64_t)blockIdx.x * CGout * 8 + cgo * 8 + threadIdx.x] = s;
  }
}

// Fixed-order reduction over splits, scatter into DHWIO fp32 (unpadded channels).
__global__ void k_wgrad_finalize(const float* __restrict__ ws, const float* __restrict__ wsb,
                                 float* __restrict__ gw, float* __restrict__ gb, int nsplit,
                                 int Cin, int Cout, int CGin, int CGout) {
  const int64_t n = (int64_t)27 * Cin * Cout;
  const int64_t stride_split = (int64_t)27 * CGin * 8 * CGout * 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + Cout;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      int co = i % Cout;
      int ci = (i / Cout) % Cin;
      int t = (int)(i / ((int64_t)Cout * Cin));
      int64_t src = ((int64_t)t * CGin * 8 + ci) * CGout * 8 + co;
      float s = 0.f;
      for (int sp = 0; sp < nsplit; ++sp) s += ws[sp * stride_split + src];
      gw[i] = s;
    } else {
      int co = (int)(i - n);
      float s = 0.f;
      for (int sp = 0; sp < nsplit; ++sp) s += wsb[(int64_t)sp * CGout * 8 + co];
      gb[co] = s;
    }
  }
}

__global__ void k_flip_transpose(const float* __restrict__ w, float* __restrict__ wt, int k,
                                 int Cin, int Cout) {
  const int T = k * k * k;
  const int64_t n = (int64_t)T * Cin * Cout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // wt[t'][co][ci] = w[T-1-t'][ci][co]
    int ci = i % Cin;
    int co = (i / Cin) % Cout;
    int tp = (int)(i / ((int64_t)Cin * Cout));
    wt[i] = w[((int64_t)(T - 1 - tp) * Cin + ci) * Cout + co];
  }
}

__global__ void k_bias_finalize(const float* __restrict__ wsb, float* __restrict__ gb, int nsplit,
                                int Cout, int CGout) {
  for (int co = blockIdx.x * blockDim.x + threadIdx.x; co < Cout; co += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) s += wsb[(int64_t)sp * CGout * 8 + co];
    gb[co] = s;
  }
}

size_t bias_grad_ws_bytes(int64_t nvox, int Cout) {
  int64_t s = nvox / 1024;  // ~4 voxels per thread per block
  if (s < 1) s = 1;
  if (s > 512) s = 512;
  return (size_t)s * ((Cout + 7) / 8) * 8 * sizeof(float);
}

// Per-split partial sums of gy over interior voxels: ws[ns][CGo*8] (bf16 slab); the caller
// reduces the ns splits in order.
int bias_grad_partial_bf16(const void* gy, int64_t gy_bstride, float* ws, int B, int Cout, int D, int H, int W,
                           cudaStream_t st, int* nsplit) {
  const Slab gg = make_slab(gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1), (Cout + 7) / 8, D, H, W, 1);
  int64_t nvox = (int64_t)B * D * H * W;
  VM_REQUIRE(nvox < (1LL << 31), VM_E_SHAPE, "bias_grad_partial_bf16: %lld voxels", (long long)nvox);
  int ns = (int)(bias_grad_ws_bytes(nvox, Cout) / (gg.CG * 8 * sizeof(float)));
  int64_t chunk = (nvox + ns - 1) / ns;
  launch_pdl(k_bias_grad_partial<__nv_bfloat16>, dim3(ns, gg.CG), 256, 0, st, (const __nv_bfloat16*)gy, gg, ws, B,
             gg.CG, chunk);
  *nsplit = ns;
  return launch_status("bias_grad_partial_bf16");
}

// gb[co] = sum over interior voxels of gy[.., co], deterministic (bf16 slab)
int bias_grad_bf16(const void* gy, int64_t gy_bstride, float* gb, float* ws, int B, int Cout, int D,
                   int H, int W, cudaStream_t st) {
  const Slab gg = make_slab(gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1), (Cout + 7) / 8, D, H, W, 1);
  int64_t nvox = (int64_t)B * D * H * W;
  VM_REQUIRE(nvox < (1LL << 31), VM_E_SHAPE, "bias_grad_bf16: %lld voxels", (long long)nvox);
  int ns = (int)(bias_grad_ws_bytes(nvox, Cout) / (gg.CG * 8 * sizeof(float)));
  int64_t chunk = (nvox + ns - 1) / ns;
  k_bias_grad_partial<__nv_bfloat16><<<dim3(ns, gg.CG), 256, 0, st>>>((const __nv_bfloat16*)gy, gg, ws, B,
                                                                      gg.CG, chunk);
  k_bias_finalize<<<1, 128, 0, st>>>(ws, gb, ns, Cout, gg.CG);
  return launch_status("bias_grad_bf16", 2);
}

static int wgrad_splits(int64_t nvox, int64_t combos) {
  int64_t s = nvox / 4096;
  if (s < 1) s = 1;
  if (s > 64) s = 64;
  while (s > 1 && s * combos > 65535 * 4) s /= 2;
  return (int)s;
}

}  // namespace vm

using namespace vm;

extern "C" int vm_conv3d_fwd_simt(int dtype, const void* x, int64_t x_bstride, const float* w,
                                  const float* bias, void* y, int64_t y_bstride, const void* mask,
                                  int64_t mask_bstride, int B, int Cin, int Cout, int D, int H, int W,
                                  unsigned flags, void* stream) {
  VM_REQUIRE(x && w && y, VM_E_ARG, "vm_conv3d_fwd_simt: null pointer");
  VM_REQUIRE((flags & VM_CONV_NOBIAS) || bias, VM_E_ARG, "vm_conv3d_fwd_simt: bias required");
  VM_REQUIRE(!(flags & VM_CONV_MASK) || mask, VM_E_ARG, "vm_conv3d_fwd_simt: mask required");
  VM_REQUIRE(B > 0 && Cin > 0 && Cout > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE,
             "vm_conv3d_fwd_simt: bad shape");
  Slab gx{x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1), (Cin + 7) / 8, D, H, W, 1};
  Slab gy{y_bstride ? y_bstride : default_bstride(Cout, D, H, W, 1), (Cout + 7) / 8, D, H, W, 1};
  Slab gm{mask_bstride ? mask_bstride : default_bstride(Cout, D, H, W, 1), (Cout + 7) / 8, D, H, W, 1};
  int64_t nvox = (int64_t)B * D * H * W;
  dim3 grid((unsigned)((nvox + 127) / 128), (unsigned)gy.CG);
  cudaStream_t st = as_stream(stream);
  if (dtype == VM_F32)
    k_conv_fwd_simt<float><<<grid, 128, 0, st>>>((const float*)x, gx, w, bias, (float*)y, gy,
                                                  (const float*)mask, gm, B, Cin, Cout, flags);
  else if (dtype == VM_BF16)
    k_conv_fwd_simt<__nv_bfloat16><<<grid, 128, 0, st>>>(
        (const __nv_bfloat16*)x, gx, w, bias, (__nv_bfloat16*)y, gy, (const __nv_bfloat16*)mask,
        gm, B, Cin, Cout, flags);
  else
    VM_REQUIRE(false, VM_E_DTYPE, "vm_conv3d_fwd_simt: dtype %d", dtype);
  return launch_status("vm_conv3d_fwd_simt");
}

extern "C" size_t vm_conv3d_wgrad_simt_ws(int B, int Cin, int Cout, int D, int H, int W) {
  int64_t nvox = (int64_t)B * D * H * W;
  int CGin = (Cin + 7) / 8, CGout = (Cout + 7) / 8;
  int ns = wgrad_splits(nvox, (int64_t)27 * CGin * CGout);
  return (size_t)ns * 27 * CGin * 8 * CGout * 8 * 4 + (size_t)ns * CGout * 8 * 4;
}

extern "C" int vm_conv3d_wgrad_simt(int dtype, const void* x, int64_t x_bstride, const void* gy,
                                    int64_t gy_bstride, float* gw, float* gb, void* ws, int B,
                                    int Cin, int Cout, int D, int H, int W, void* stream) {
  VM_REQUIRE(x && gy && gw && gb && ws, VM_E_ARG, "vm_conv3d_wgrad_simt: null pointer");
  VM_REQUIRE(B > 0 && Cin > 0 && Cout > 0 && D > 0 && H > 0 && W > 0, VM_E_SHAPE,
             "vm_conv3d_wgrad_simt: bad shape");
  Slab gx{x_bstride ? x_bstride : default_bstride(Cin, D, H, W, 1), (Cin + 7) / 8, D, H, W, 1};
  const Slab gg = make_slab(gy_bstride ? gy_bstride : default_bstride(Cout, D, H, W, 1), (Cout + 7) / 8, D, H, W, 1);
  int64_t nvox = (int64_t)B * D * H * W;
  int CGin = gx.CG, CGout = gg.CG;
  int ns = wgrad_splits(nvox, (int64_t)27 * CGin * CGout);
  int64_t chunk = (nvox + ns - 1) / ns;
  float* wsw = static_cast<float*>(ws);
  float* wsb = wsw + (size_t)ns * 27 * CGin * 8 * CGout * 8;
  cudaStream_t st = as_stream(stream);
  dim3 grid(27 * CGin * CGout, ns);
  dim3 gridb(ns, CGout);
  if (dtype == VM_F32) {
    k_conv_wgrad_simt<float><<<grid, 256, 0, st>>>((const float*)x, gx, (const float*)gy, gg, wsw,
                                                    B, CGin, CGout, chunk);
    k_bias_grad_partial<float><<<gridb, 256, 0, st>>>((const float*)gy, gg, wsb, B, CGout, chunk);
  } else if (dtype == VM_BF16) {
    k_conv_wgrad_simt<__nv_bfloat16><<<grid, 256, 0, st>>>(
        (const __nv_bfloat16*)x, gx, (const __nv_bfloat16*)gy, gg, wsw, B, CGin, CGout, chunk);
    k_bias_grad_partial<__nv_bfloat16><<<gridb, 256, 0, st>>>((const __nv_bfloat16*)gy, gg, wsb, B,
                                                             CGout, chunk);
  } else {
    VM_REQUIRE(false, VM_E_DTYPE, "vm_conv3d_wgrad_simt: dtype %d", dtype);
  }
  k_wgrad_finalize<<<grid_for((int64_t)27 * Cin * Cout + Cout, 256), 256, 0, st>>>(
      wsw, wsb, gw, gb, ns, Cin, Cout, CGin, CGout);
  return launch_status("vm_conv3d_wgrad_simt", 3);
}

extern "C" int vm_weight_flip_transpose(const float* w, float* wt, int k, int Cin, int Cout,
                                        void* stream) {
  VM_REQUIRE(w && wt && k > 0 && Cin > 0 && Cout > 0, VM_E_ARG, "vm_weight_flip_transpose: bad arg");
  k_flip_transpose<<<grid_for((int64_t)k * k * k * Cin * Cout, 256), 256, 0, as_stream(stream)>>>(
      w, wt, k, Cin, Cout);
  return launch_status("vm_weight_flip_transpose");
}
