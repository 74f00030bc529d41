// pointwise.cu — HBM-bound kernels of the step on channel-blocked slabs:
// maxpool2 fwd/bwd, nearest upsample x2 fwd/bwd, relu mask, fused head
// (1x1x1 conv + softmax + Dice/CE statistics and gradient), fixed-order
// reductions, SGD with momentum.  One 16-byte channel-block vector per thread
// access; grids are multiples of the SM count (grid-stride loops).
#include <cfloat>

#include "vm_common.cuh"

namespace vm {

template <typename T> struct V8;
template <> struct V8<float> {
  __device__ __forceinline__ static void ld(const float* p, float (&v)[8]) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ __forceinline__ static void st(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <> struct V8<__nv_bfloat16> {
  __device__ __forceinline__ static void ld(const __nv_bfloat16* p, float (&v)[8]) {
    int4 raw = *reinterpret_cast<const int4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  }
  __device__ __forceinline__ static void st(__nv_bfloat16* p, const float (&v)[8]) {
    int4 raw;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<int4*>(p) = raw;
  }
};

// 32-bit index math: every launch checks that its index space fits (vm_fits32); 64-bit
// division costs ~4x the instructions and these kernels are issue-bound at HBM speed
__device__ __forceinline__ void decompose(uint32_t v, const Slab& s, int& b, int& d, int& h, int& w) {
  const uint32_t q1 = fastdiv(v, (uint32_t)s.W, s.mW);
  w = (int)(v - q1 * (uint32_t)s.W);
  const uint32_t q2 = fastdiv(q1, (uint32_t)s.H, s.mH);
  h = (int)(q1 - q2 * (uint32_t)s.H);
  const uint32_t q3 = fastdiv(q2, (uint32_t)s.D, s.mD);
  d = (int)(q2 - q3 * (uint32_t)s.D);
  b = (int)q3;
}
__device__ __forceinline__ int split_cg(int64_t i, int64_t nvox, uint32_t& v) {
  const uint32_t i32 = (uint32_t)i, n32 = (uint32_t)nvox;
  const uint32_t cg = i32 / n32;
  v = i32 - cg * n32;
  return (int)cg;
}

// ------------------------------------------------------------------ maxpool
// out grid: pooled voxels (D,H,W are the POOLED extents) x channel blocks
template <typename T>
__global__ void k_maxpool_fwd(const T* __restrict__ x, Slab gx, T* __restrict__ y, Slab gy, int B) {
  pdl_wait();
  pdl_trigger();
  const int64_t nvox = (int64_t)B * gy.D * gy.H * gy.W;
  const int64_t total = nvox * gy.CG;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v32;
    int cg = split_cg(i, nvox, v32);
    int b, d, h, w;
    decompose(v32, gy, b, d, h, w);
    float best[8];
    for (int cell = 0; cell < 8; ++cell) {  // (dz, dy, dx) scan order, ops.py:149-154
      float v[8];
      V8<T>::ld(x + gx.at(b, cg, 2 * d + (cell >> 2), 2 * h + ((cell >> 1) & 1), 2 * w + (cell & 1)), v);
#pragma unroll
      for (int j = 0; j < 8; ++j) best[j] = (cell == 0 || v[j] > best[j]) ? v[j] : best[j];
    }
    V8<T>::st(y + gy.at(b, cg, d, h, w), best);
  }
}

// gin[cell] = (cell == argmax) ? gout : 0, first max wins (np.argmax), + add, * (x>0)
template <typename T>
__global__ void k_maxpool_bwd(const T* __restrict__ x, Slab gx, const T* __restrict__ gout, Slab go,
                              const T* __restrict__ add, Slab ga, T* __restrict__ gin, Slab gi,
                              int B, int relu_mask) {
  pdl_wait();
  const int64_t nvox = (int64_t)B * go.D * go.H * go.W;
  const int64_t total = nvox * go.CG;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v32;
    int cg = split_cg(i, nvox, v32);
    int b, d, h, w;
    decompose(v32, go, b, d, h, w);
    // one pass over the 2x2x2 cell: argmax per channel (first max wins) and the ReLU mask
    // bits (x > 0) per (cell, channel), so the write pass needs no second read of x
    int arg[8];
    float best[8];
    uint32_t pos_lo = 0, pos_hi = 0;  // bit (cell*8 + j): x > 0
#pragma unroll
    for (int cell = 0; cell < 8; ++cell) {
      float xv[8];
      V8<T>::ld(x + gx.at(b, cg, 2 * d + (cell >> 2), 2 * h + ((cell >> 1) & 1), 2 * w + (cell & 1)), xv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (cell == 0 || xv[j] > best[j]) {
          best[j] = xv[j];
          arg[j] = cell;
        }
        if (xv[j] > 0.f) {
          if (cell < 4) pos_lo |= 1u << (cell * 8 + j);
          else pos_hi |= 1u << ((cell - 4) * 8 + j);
        }
      }
    }
    float g[8];
    V8<T>::ld(gout + go.at(b, cg, d, h, w), g);
#pragma unroll 2
    for (int cell = 0; cell < 8; ++cell) {
      int pd = 2 * d + (cell >> 2), ph = 2 * h + ((cell >> 1) & 1), pw = 2 * w + (cell & 1);
      float o[8];
      if (add) V8<T>::ld(add + ga.at(b, cg, pd, ph, pw), o);
      const uint32_t pos = cell < 4 ? pos_lo >> (cell * 8) : pos_hi >> ((cell - 4) * 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float r = (arg[j] == cell) ? g[j] : 0.f;
        if (add) r += o[j];
        if (relu_mask && !((pos >> j) & 1u)) r = 0.f;
        o[j] = r;
      }
      V8<T>::st(gin + gi.at(b, cg, pd, ph, pw), o);
    }
  }
}

// ------------------------------------------------------------------ upsample
// two threads per INPUT channel-block vector (one per output w parity): one load, then the
// vector goes to the four (dz, dy) rows of the 2x2x2 output cell.  A warp's store instruction
// writes 32 consecutive output vectors (512 contiguous bytes); the index decomposition runs
// once per 4 outputs instead of once per output (that version was issue-bound at ~3.4 TB/s,
// and one thread per input writing 16 B at a 32 B lane stride measured slower still).
template <typename T>
__global__ void k_upsample_fwd(const T* __restrict__ x, Slab gx, T* __restrict__ y, Slab gy, int B) {
  pdl_wait();
  pdl_trigger();
  const int64_t nvox = (int64_t)B * gx.D * gx.H * gx.W;
  const int64_t total = nvox * gx.CG * 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int par = (int)(i & 1);
    uint32_t v32;
    int cg = split_cg(i >> 1, nvox, v32);
    int b, d, h, w;
    decompose(v32, gx, b, d, h, w);
    const T* src = x + gx.at(b, cg, d, h, w);
    const int4 a0 = __ldg(reinterpret_cast<const int4*>(src));
    const int4 a1 = sizeof(T) == 4 ? __ldg(reinterpret_cast<const int4*>(src + 4)) : a0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int4* o = reinterpret_cast<int4*>(y + gy.at(b, cg, 2 * d + (r >> 1), 2 * h + (r & 1), 2 * w + par));
      o[0] = a0;
      if (sizeof(T) == 4) o[1] = a1;
    }
  }
}

template <typename T>
__global__ void k_upsample_bwd(const T* __restrict__ gy, Slab sgy, const T* __restrict__ mask,
                               Slab sm, T* __restrict__ gx, Slab sgx, int B) {
  pdl_wait();
  const int64_t nvox = (int64_t)B * sgx.D * sgx.H * sgx.W;
  const int64_t total = nvox * sgx.CG;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v32;
    int cg = split_cg(i, nvox, v32);
    int b, d, h, w;
    decompose(v32, sgx, b, d, h, w);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int cell = 0; cell < 8; ++cell) {
      float v[8];
      V8<T>::ld(gy + sgy.at(b, cg, 2 * d + (cell >> 2), 2 * h + ((cell >> 1) & 1), 2 * w + (cell & 1)), v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
    if (mask) {
      float mv[8];
      V8<T>::ld(mask + sm.at(b, cg, d, h, w), mv);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = mv[j] > 0.f ? acc[j] : 0.f;
    }
    V8<T>::st(gx + sgx.at(b, cg, d, h, w), acc);
  }
}

template <typename T>
__global__ void k_relu_mask(const T* __restrict__ g, Slab sg, const T* __restrict__ mask, Slab sm,
                            T* __restrict__ out, Slab so, int B) {
  const int64_t nvox = (int64_t)B * sg.D * sg.H * sg.W;
  const int64_t total = nvox * sg.CG;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v32;
    int cg = split_cg(i, nvox, v32);
    int b, d, h, w;
    decompose(v32, sg, b, d, h, w);
    float v[8], mv[8];
    V8<T>::ld(g + sg.at(b, cg, d, h, w), v);
    V8<T>::ld(mask + sm.at(b, cg, d, h, w), mv);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = mv[j] > 0.f ? v[j] : 0.f;
    V8<T>::st(out + so.at(b, cg, d, h, w), v);
  }
}

// ------------------------------------------------------------------ head + loss
constexpr int kHeadThreads = 256;
constexpr int kMaxCls = 8;

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x == 0)
    for (int i = 0; i < kHeadThreads / 32; ++i) s += red[i];
  return s;  // valid in thread 0
}

template <typename T>
__device__ __forceinline__ void head_logits(const T* __restrict__ y, Slab sy, int b, int d, int h,
                                            int w, const float* sW, const float* sb, int C,
                                            int ncls, float* logits) {
  for (int k = 0; k < ncls; ++k) logits[k] = sb[k];
  for (int cg = 0; cg < sy.CG; ++cg) {
    float v[8];
    V8<T>::ld(y + sy.at(b, cg, d, h, w), v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int c = cg * 8 + j;
      if (c < C)
        for (int k = 0; k < ncls; ++k) logits[k] = fmaf(v[j], sW[c * ncls + k], logits[k]);
    }
  }
}

__device__ __forceinline__ void softmax_n(const float* logits, int ncls, float* p) {
  float m = logits[0];
  for (int k = 1; k < ncls; ++k) m = fmaxf(m, logits[k]);
  float s = 0.f;
  for (int k = 0; k < ncls; ++k) {
    p[k] = expf(logits[k] - m);
    s += p[k];
  }
  for (int k = 0; k < ncls; ++k) p[k] = p[k] / s;
}

template <typename T>
__global__ void __launch_bounds__(kHeadThreads) k_head_fwd(const T* __restrict__ y, Slab sy,
                                                           const float* __restrict__ W,
                                                           const float* __restrict__ bias,
                                                           const uint8_t* __restrict__ labels,
                                                           int* __restrict__ label_err,
                                                           float* __restrict__ probs,
                                                           uint8_t* __restrict__ pred,
                                                           float* __restrict__ partials, int B,
                                                           int C, int ncls, float clamp) {
  extern __shared__ float sh[];
  float* sW = sh;
  float* sb = sW + C * ncls;
  float* red = sb + ncls;
  for (int i = threadIdx.x; i < C * ncls; i += blockDim.x) sW[i] = W[i];
  for (int i = threadIdx.x; i < ncls; i += blockDim.x) sb[i] = bias[i];
  __syncthreads();
  const int64_t nvox = (int64_t)B * sy.D * sy.H * sy.W;
  float st[3 * kMaxCls + 1];
  for (int k = 0; k < 3 * ncls + 1; ++k) st[k] = 0.f;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
       v += (int64_t)gridDim.x * blockDim.x) {
    int b, d, h, w;
    decompose((uint32_t)v, sy, b, d, h, w);
    float lg[kMaxCls], p[kMaxCls];
    head_logits(y, sy, b, d, h, w, sW, sb, C, ncls, lg);
    softmax_n(lg, ncls, p);
    if (labels[v] >= ncls) atomicOr(label_err, 1);
    if (pred) {  // np.argmax: the first maximal class
      int a = 0;
      for (int k = 1; k < ncls; ++k) a = p[k] > p[a] ? k : a;
      pred[v] = (uint8_t)a;
    }
    for (int k = 0; k < ncls; ++k) {
      const float g = labels[v] == k ? 1.f : 0.f;
      if (probs) probs[v * ncls + k] = p[k];
      st[k] += p[k] * g;
      st[ncls + k] += p[k];
      st[2 * ncls + k] += g;
      st[3 * ncls] += -logf(fmaxf(p[k], clamp)) * g;
    }
  }
  for (int k = 0; k < 3 * ncls + 1; ++k) {
    float s = block_sum(st[k], red);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.x * (3 * ncls + 1) + k] = s;
  }
}

template <typename T>
__global__ void __launch_bounds__(kHeadThreads) k_head_bwd(
    const T* __restrict__ y, Slab sy, const float* __restrict__ W, const float* __restrict__ bias,
    const uint8_t* __restrict__ labels, const float* __restrict__ stats, T* __restrict__ g, Slab sg,
    float* __restrict__ wpart, int B, int C, int ncls, float w_dice, float w_ce, float total,
    int dice_mask, float clamp, int relu_mask, const float* __restrict__ dprobs) {
  extern __shared__ float sh[];
  float* sW = sh;
  float* sb = sW + C * ncls;
  float* red = sb + ncls;
  float* coef = red + 32;  // per class: a_k (dice slope), r_k (dice ratio), active flag
  for (int i = threadIdx.x; i < C * ncls; i += blockDim.x) sW[i] = W[i];
  for (int i = threadIdx.x; i < ncls; i += blockDim.x) sb[i] = bias[i];
  if (threadIdx.x == 0) {
    int nfg = __popc(dice_mask);
    for (int k = 0; k < ncls; ++k) {
      // training.py:119-124 — grad_k += (-w_d/nfg) * (2 g_k - r_k) / d_k
      float nk = stats ? 2.f * stats[k] + 1e-6f : 1.f;
      float dk = stats ? stats[ncls + k] + stats[2 * ncls + k] + 1e-6f : 1.f;
      bool on = (dice_mask >> k) & 1;
      coef[3 * k + 0] = on ? (-w_dice / (float)nfg) / dk : 0.f;
      coef[3 * k + 1] = on ? nk / dk : 0.f;
      coef[3 * k + 2] = on ? 1.f : 0.f;
    }
  }
  __syncthreads();
  const int64_t nvox = (int64_t)B * sy.D * sy.H * sy.W;
  const float ce_scale = -w_ce / total;
  // per-thread weight-grad partials: sum_v y_c * gl_k (C*ncls) + sum_v gl_k (ncls)
  // accumulated per channel block to bound registers; C*ncls <= 64*8 handled by loop
  const int nw = C * ncls + ncls;
  for (int base = 0; base < nw; base += 64) {
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0.f;
    const bool write_g = (base == 0);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
         v += (int64_t)gridDim.x * blockDim.x) {
      int b, d, h, w;
      decompose((uint32_t)v, sy, b, d, h, w);
      float lg[kMaxCls], p[kMaxCls], gp[kMaxCls], gl[kMaxCls];
      head_logits(y, sy, b, d, h, w, sW, sb, C, ncls, lg);
      softmax_n(lg, ncls, p);
      float dot = 0.f;
      for (int k = 0; k < ncls; ++k) {
        const float gk = labels && labels[v] == k ? 1.f : 0.f;
        float r = coef[3 * k + 2] != 0.f ? coef[3 * k] * (2.f * gk - coef[3 * k + 1]) : 0.f;
        float pm = fmaxf(p[k], clamp);
        r += p[k] >= clamp ? ce_scale * (gk / pm) : 0.f;  // training.py:125-126
        if (dprobs) r = dprobs[v * ncls + k];  // external dL/dp (run_backward_local)
        gp[k] = r;
        dot += r * p[k];
      }
      for (int k = 0; k < ncls; ++k) gl[k] = p[k] * (gp[k] - dot);  // ops.py:197-199
      for (int cg = 0; cg < sy.CG; ++cg) {
        float yv[8];
        V8<T>::ld(y + sy.at(b, cg, d, h, w), yv);
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          int c = cg * 8 + j;
          float s = 0.f;
          if (c < C) {
            for (int k = 0; k < ncls; ++k) {
              s = fmaf(sW[c * ncls + k], gl[k], s);
              int idx = c * ncls + k - base;
              if (idx >= 0 && idx < 64) acc[idx] = fmaf(yv[j], gl[k], acc[idx]);
            }
          }
          o[j] = (relu_mask && !(yv[j] > 0.f)) ? 0.f : s;
        }
        if (write_g) V8<T>::st(g + sg.at(b, cg, d, h, w), o);
      }
      for (int k = 0; k < ncls; ++k) {
        int idx = C * ncls + k - base;
        if (idx >= 0 && idx < 64) acc[idx] += gl[k];
      }
    }
    for (int i = 0; i < 64 && base + i < nw; ++i) {
      float s = block_sum(acc[i], red);
      if (threadIdx.x == 0) wpart[(int64_t)blockIdx.x * nw + base + i] = s;
    }
  }
}

// Fixed-shape head kernels (C input channels, NC classes known at compile time): all
// per-voxel state and the weight-gradient partials live in registers.
template <typename T, int C, int NC>
__global__ void __launch_bounds__(kHeadThreads, 2) k_head_fwd_fixed(
    const T* __restrict__ y, Slab sy, const float* __restrict__ W, const float* __restrict__ bias,
    const uint8_t* __restrict__ labels, int* __restrict__ label_err, float* __restrict__ probs,
    uint8_t* __restrict__ pred, float* __restrict__ partials, int B, float clamp) {
  static_assert(sizeof(T) == 2, "fixed head kernels read bf16 channel groups as 16-byte words");
  pdl_wait();
  pdl_trigger();
  __shared__ float sW[C * NC], sb[NC], red[kHeadThreads / 32];
  for (int i = threadIdx.x; i < C * NC; i += blockDim.x) sW[i] = W[i];
  if (threadIdx.x < NC) sb[threadIdx.x] = bias[threadIdx.x];
  __syncthreads();
  const int64_t nvox = (int64_t)B * sy.D * sy.H * sy.W;
  float st[3 * NC + 1];
#pragma unroll
  for (int k = 0; k < 3 * NC + 1; ++k) st[k] = 0.f;
  // U voxels per thread per iteration with every load issued first (loads in flight bound
  // it): the raw 16-byte channel groups of all U voxels are loaded before any math, then the
  // logits are summed in channel order (bitwise the same as a full dot product).  (Loading
  // two groups at a time at U = 1 held C = 32 to ~0.37 of HBM.)
  constexpr int U = C <= 16 ? 2 : 1;
  constexpr int NG = C / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nvox; v0 += U * stride) {
    float lgu[U][NC], gk[U][NC];
    bool ok[U];
    int4 raw[U][C <= 32 ? NG : 1];
    uint32_t labu[U];
    const T* basep[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * stride;
      ok[u] = v < nvox;
      int b, d, h, w;
      decompose(ok[u] ? (uint32_t)v : 0u, sy, b, d, h, w);
      basep[u] = y + sy.at(b, 0, d, h, w);
      if (C <= 32) {
#pragma unroll
        for (int cg = 0; cg < (C <= 32 ? NG : 1); ++cg)
          raw[u][cg] = *reinterpret_cast<const int4*>(basep[u] + cg * sy.plane());
      }
      labu[u] = ok[u] ? labels[v] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k = 0; k < NC; ++k) lgu[u][k] = sb[k];
      if (C <= 32) {
#pragma unroll
        for (int cg = 0; cg < (C <= 32 ? NG : 1); ++cg) {
          const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&raw[u][cg]);
          float t8[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(hv[j]);
            t8[2 * j] = f.x;
            t8[2 * j + 1] = f.y;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < NC; ++k) lgu[u][k] = fmaf(t8[j], sW[(cg * 8 + j) * NC + k], lgu[u][k]);
        }
      } else {
#pragma unroll 2
        for (int cg = 0; cg < NG; ++cg) {
          float t8[8];
          V8<T>::ld(basep[u] + cg * sy.plane(), t8);
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < NC; ++k) lgu[u][k] = fmaf(t8[j], sW[(cg * 8 + j) * NC + k], lgu[u][k]);
        }
      }
      const uint32_t lab = labu[u];
      if (lab >= (uint32_t)NC) atomicOr(label_err, 1);  // training.py:68-69 (np.eye indexing) raises
#pragma unroll
      for (int k = 0; k < NC; ++k) gk[u][k] = lab == (uint32_t)k ? 1.f : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int64_t v = v0 + u * stride;
      float lg[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) lg[k] = lgu[u][k];
      float m = lg[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) m = fmaxf(m, lg[k]);
      float p[NC], ssum = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __expf(lg[k] - m);
        ssum += p[k];
      }
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __fdividef(p[k], ssum);
        const float g = gk[u][k];
        if (probs) probs[v * NC + k] = p[k];
        st[k] += p[k] * g;
        st[NC + k] += p[k];
        st[2 * NC + k] += g;
        st[3 * NC] += -__logf(fmaxf(p[k], clamp)) * g;
      }
      if (pred) {  // np.argmax of these probabilities: the first maximal class
        int a = 0;
#pragma unroll
        for (int k = 1; k < NC; ++k) a = p[k] > p[a] ? k : a;
        pred[v] = (uint8_t)a;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 3 * NC + 1; ++k) {
    float s = block_sum(st[k], red);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.x * (3 * NC + 1) + k] = s;
  }
}

template <typename T, int C, int NC>
__global__ void __launch_bounds__(kHeadThreads, 2) k_head_bwd_fixed(
    const T* __restrict__ y, Slab sy, const float* __restrict__ W, const float* __restrict__ bias,
    const uint8_t* __restrict__ labels, const float* __restrict__ stats, T* __restrict__ g, Slab sg,
    float* __restrict__ wpart, int B, float w_dice, float w_ce, float total, int dice_mask, float clamp,
    int relu_mask) {
  __shared__ float sW[C * NC], sb[NC], red[kHeadThreads / 32], coef[3 * NC];
  for (int i = threadIdx.x; i < C * NC; i += blockDim.x) sW[i] = W[i];
  if (threadIdx.x < NC) sb[threadIdx.x] = bias[threadIdx.x];
  if (threadIdx.x == 0) {
    const int nfg = __popc(dice_mask);
    for (int k = 0; k < NC; ++k) {  // training.py:119-124
      const float nk = stats ? 2.f * stats[k] + 1e-6f : 1.f;
      const float dk = stats ? stats[NC + k] + stats[2 * NC + k] + 1e-6f : 1.f;
      const bool on = (dice_mask >> k) & 1;
      coef[3 * k + 0] = on ? (-w_dice / (float)nfg) / dk : 0.f;
      coef[3 * k + 1] = on ? nk / dk : 0.f;
      coef[3 * k + 2] = on ? 1.f : 0.f;
    }
  }
  __syncthreads();
  const int64_t nvox = (int64_t)B * sy.D * sy.H * sy.W;
  const float ce_scale = -w_ce / total;
  float acc[C * NC + NC];
#pragma unroll
  for (int i = 0; i < C * NC + NC; ++i) acc[i] = 0.f;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
       v += (int64_t)gridDim.x * blockDim.x) {
    int b, d, h, w;
    decompose((uint32_t)v, sy, b, d, h, w);
    float yv[C];
    const T* base = y + sy.at(b, 0, d, h, w);
#pragma unroll
    for (int cg = 0; cg < C / 8; ++cg) {
      float t8[8];
      V8<T>::ld(base + cg * sy.plane(), t8);
#pragma unroll
      for (int j = 0; j < 8; ++j) yv[cg * 8 + j] = t8[j];
    }
    float lg[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      lg[k] = sb[k];
#pragma unroll
      for (int c = 0; c < C; ++c) lg[k] = fmaf(yv[c], sW[c * NC + k], lg[k]);
    }
    float m = lg[0];
#pragma unroll
    for (int k = 1; k < NC; ++k) m = fmaxf(m, lg[k]);
    float p[NC], ssum = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      p[k] = expf(lg[k] - m);
      ssum += p[k];
    }
    float gp[NC], dot = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      p[k] = p[k] / ssum;
      const float gk = labels[v] == k ? 1.f : 0.f;
      float r = coef[3 * k + 2] != 0.f ? coef[3 * k] * (2.f * gk - coef[3 * k + 1]) : 0.f;
      r += p[k] >= clamp ? ce_scale * (gk / fmaxf(p[k], clamp)) : 0.f;  // training.py:125-126
      gp[k] = r;
      dot += r * p[k];
    }
    float gl[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      gl[k] = p[k] * (gp[k] - dot);  // ops.py:197-199
      acc[C * NC + k] += gl[k];
    }
    T* gbase = g + sg.at(b, 0, d, h, w);
#pragma unroll
    for (int cg = 0; cg < C / 8; ++cg) {
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = cg * 8 + j;
        float sacc = 0.f;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          sacc = fmaf(sW[c * NC + k], gl[k], sacc);
          acc[c * NC + k] = fmaf(yv[c], gl[k], acc[c * NC + k]);
        }
        o[j] = (relu_mask && !(yv[c] > 0.f)) ? 0.f : sacc;
      }
      V8<T>::st(gbase + cg * sg.plane(), o);
    }
  }
#pragma unroll
  for (int i = 0; i < C * NC + NC; ++i) {
    float s = block_sum(acc[i], red);
    if (threadIdx.x == 0) wpart[(int64_t)blockIdx.x * (C * NC + NC) + i] = s;
  }
}

// Head backward with C/8 threads per voxel (one 8-channel group each): logits are summed
// across the group with shuffles, so a thread holds 8*NC (+NC) weight-gradient accumulators
// instead of C*NC + NC (no spills, full occupancy).  Per-block partials are reduced over lanes
// of the same group and then over warps in a fixed order (deterministic), into the layout
// of k_head_bwd_fixed: wpart[block][c*NC + k], bias at [C*NC + k].
template <typename T, int C, int NC>
__global__ void __launch_bounds__(kHeadThreads, 2) k_head_bwd_grp(
    const T* __restrict__ y, Slab sy, const float* __restrict__ W, const float* __restrict__ bias,
    const uint8_t* __restrict__ labels, const float* __restrict__ stats, T* __restrict__ g, Slab sg,
    float* __restrict__ wpart, int B, float w_dice, float w_ce, float total, int dice_mask, float clamp,
    int relu_mask, const float* __restrict__ dprobs) {
  pdl_wait();
  constexpr int TPV = C / 8;
  constexpr int NACC = 8 * NC + NC;  // group's weight grads + bias grads (used by cg == 0)
  constexpr int NWARP = kHeadThreads / 32;
  __shared__ float sW[C * NC], sb[NC], coef[3 * NC];
  __shared__ float red[NWARP][TPV][NACC];
  for (int i = threadIdx.x; i < C * NC; i += blockDim.x) sW[i] = W[i];
  if (threadIdx.x < NC) sb[threadIdx.x] = bias[threadIdx.x];
  if (threadIdx.x == 0) {
    const int nfg = __popc(dice_mask);
    for (int k = 0; k < NC; ++k) {  // training.py:119-124
      const float nk = stats ? 2.f * stats[k] + 1e-6f : 1.f;
      const float dk = stats ? stats[NC + k] + stats[2 * NC + k] + 1e-6f : 1.f;
      const bool on = (dice_mask >> k) & 1;
      coef[3 * k + 0] = on ? (-w_dice / (float)nfg) / dk : 0.f;
      coef[3 * k + 1] = on ? nk / dk : 0.f;
      coef[3 * k + 2] = on ? 1.f : 0.f;
    }
  }
  __syncthreads();
  const int cg = threadIdx.x % TPV;
  // this thread's 8 channels of the head weights, read from shared memory (two broadcast
  // addresses per warp): keeping them in registers left room for only 2 items in flight
  const float* wr = sW + cg * 8 * NC;
  const uint32_t nvox = (uint32_t)B * sy.D * sy.H * sy.W;
  const float ce_scale = -w_ce / total;
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.f;
  // U voxel items per thread per iteration, all loads issued before any math: the kernel is
  // limited by loads in flight (2 blocks of 256 threads per SM), not by arithmetic
  constexpr int U = 3;
  const uint32_t total_items = nvox * TPV;
  const uint32_t stride = gridDim.x * blockDim.x;
  // warp-uniform trip count (the loop body shuffles): iterate while the warp's first item is live
  const uint32_t lane_off = threadIdx.x & 31;
  for (uint32_t gi0 = blockIdx.x * blockDim.x + threadIdx.x; gi0 - lane_off < total_items; gi0 += U * stride) {
    float yv[U][8], gk[U][NC];
    int64_t go[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t gi = gi0 + u * stride;
      ok[u] = gi < total_items;
      const uint32_t v = ok[u] ? gi / TPV : 0u;
      int b, d, h, w;
      decompose(v, sy, b, d, h, w);
      V8<T>::ld(y + sy.at(b, cg, d, h, w), yv[u]);
      go[u] = sg.at(b, cg, d, h, w);
#pragma unroll
      for (int k = 0; k < NC; ++k) gk[u][k] = labels && labels[v] == k ? 1.f : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // (inactive tail items still run the shuffles with their lanes, then skip the store)
      float lg[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        float t = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) t = fmaf(yv[u][j], wr[j * NC + k], t);
#pragma unroll
        for (int o = 1; o < TPV; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        lg[k] = t + sb[k];
      }
      float m = lg[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) m = fmaxf(m, lg[k]);
      float p[NC], ssum = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __expf(lg[k] - m);
        ssum += p[k];
      }
      float gp[NC], dot = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __fdividef(p[k], ssum);
        float r = coef[3 * k + 2] != 0.f ? coef[3 * k] * (2.f * gk[u][k] - coef[3 * k + 1]) : 0.f;
        // g / max(p, clamp) with the correctly rounded reciprocal: exact for one-hot g in {0, 1}
        // and no division slow path (FCHK + branches showed in the stall profile)
        r += p[k] >= clamp ? ce_scale * (gk[u][k] * __frcp_rn(fmaxf(p[k], clamp))) : 0.f;  // training.py:125-126
        if (dprobs) r = ok[u] ? dprobs[(size_t)((gi0 + u * stride) / TPV) * NC + k] : 0.f;  // external dL/dp
        gp[k] = r;
        dot += r * p[k];
      }
      float gl[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) gl[k] = ok[u] ? p[k] * (gp[k] - dot) : 0.f;  // ops.py:197-199
      if (cg == 0) {
#pragma unroll
        for (int k = 0; k < NC; ++k) acc[8 * NC + k] += gl[k];
      }
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float sacc = 0.f;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          sacc = fmaf(wr[j * NC + k], gl[k], sacc);
          acc[j * NC + k] = fmaf(yv[u][j], gl[k], acc[j * NC + k]);
        }
        o[j] = (relu_mask && !(yv[u][j] > 0.f)) ? 0.f : sacc;
      }
      if (ok[u]) V8<T>::st(g + go[u], o);
    }
  }
  // reduce over the lanes of this warp holding the same group, then over warps (fixed order)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    float t = acc[i];
#pragma unroll
    for (int o = TPV; o < 32; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane < TPV) red[warp][lane][i] = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C * NC + NC; i += blockDim.x) {
    float t = 0.f;
    if (i < C * NC) {
      const int c = i / NC, k = i % NC;
      for (int wq = 0; wq < NWARP; ++wq) t += red[wq][c / 8][(c % 8) * NC + k];
    } else {
      for (int wq = 0; wq < NWARP; ++wq) t += red[wq][0][8 * NC + (i - C * NC)];
    }
    wpart[(int64_t)blockIdx.x * (C * NC + NC) + i] = t;
  }
}

// Team reduce-scatter of per-lane logit partials pl[u][k] (u < TPV voxels, this lane's 8
// channels): lane cg of the team ends with the full logits of voxel u = cg.
template <int TPV, int NC>
__device__ __forceinline__ void team_reduce_scatter(const float (&pl)[TPV][NC], int cg, float (&lg)[NC]) {
  if (TPV == 2) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const float keep = cg ? pl[1][k] : pl[0][k], send = cg ? pl[0][k] : pl[TPV - 1][k];
      lg[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
  } else {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const bool hi = cg & 2;
      const float k0 = (hi ? pl[2 % TPV][k] : pl[0][k]) + __shfl_xor_sync(0xffffffffu, hi ? pl[0][k] : pl[2 % TPV][k], 2);
      const float k1 = (hi ? pl[3 % TPV][k] : pl[1][k]) + __shfl_xor_sync(0xffffffffu, hi ? pl[1][k] : pl[3 % TPV][k], 2);
      const bool odd = cg & 1;
      lg[k] = (odd ? k1 : k0) + __shfl_xor_sync(0xffffffffu, odd ? k0 : k1, 1);
    }
  }
}

// Head forward for C = 16 / 32 on rows whose width is a multiple of 32: the team layout of
// k_head_bwd_team (TPV = C/8 lanes per TPV voxels, one 8-channel group per lane, 8*NC weights
// per lane), so every lane issues TPV (x2 at C = 16) 16-byte loads before any math and the
// softmax / statistics run once per voxel.  The one-thread-per-voxel kernel hoisted all C*NC
// weights into registers and spilled at C = 32 (~0.45 of HBM).
template <typename T, int C, int NC>
__global__ void __launch_bounds__(kHeadThreads, 2) k_head_fwd_team(
    const T* __restrict__ y, Slab sy, const float* __restrict__ W, const float* __restrict__ bias,
    const uint8_t* __restrict__ labels, int* __restrict__ label_err, float* __restrict__ probs,
    uint8_t* __restrict__ pred, float* __restrict__ partials, int B, float clamp) {
  static_assert(C == 16 || C == 32, "team kernel: C = 16 or 32");
  pdl_wait();
  pdl_trigger();
  constexpr int TPV = C / 8, TW = 32 / TPV, NWARP = kHeadThreads / 32;
  constexpr int CH = TPV == 2 ? 2 : 1;
  __shared__ float sW[C * NC], sb[NC], red[NWARP];
  for (int i = threadIdx.x; i < C * NC; i += blockDim.x) sW[i] = W[i];
  if (threadIdx.x < NC) sb[threadIdx.x] = bias[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane % TPV, team = lane / TPV;
  float wr[8 * NC];
#pragma unroll
  for (int i = 0; i < 8 * NC; ++i) wr[i] = sW[cg * 8 * NC + i];
  float st[3 * NC + 1];
#pragma unroll
  for (int k = 0; k < 3 * NC + 1; ++k) st[k] = 0.f;
  const uint32_t nchunk = (uint32_t)B * sy.D * sy.H * (sy.W / 32);
  const uint32_t wstride = gridDim.x * NWARP;
  for (uint32_t ch0 = blockIdx.x * NWARP + warp; ch0 < nchunk; ch0 += CH * wstride) {
    float yv[CH][TPV][8];
    uint32_t vme[CH];
    uint32_t lab[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t ch = min(ch0 + c * wstride, nchunk - 1);
      const uint32_t v0 = ch * 32;
      int b, d, h, w0;
      decompose(v0, sy, b, d, h, w0);
      const int64_t yo = sy.at(b, cg, d, h, w0 + team);
#pragma unroll
      for (int u = 0; u < TPV; ++u) V8<T>::ld(y + yo + (int64_t)u * TW * 8, yv[c][u]);
      vme[c] = v0 + cg * TW + team;
      lab[c] = labels[vme[c]];
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (ch0 + c * wstride >= nchunk) break;  // warp-uniform
      float pl[TPV][NC];
#pragma unroll
      for (int u = 0; u < TPV; ++u)
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          float t = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) t = fmaf(yv[c][u][j], wr[j * NC + k], t);
          pl[u][k] = t;
        }
      float lg[NC];
      team_reduce_scatter<TPV, NC>(pl, cg, lg);
#pragma unroll
      for (int k = 0; k < NC; ++k) lg[k] += sb[k];
      float m = lg[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) m = fmaxf(m, lg[k]);
      float p[NC], ssum = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __expf(lg[k] - m);
        ssum += p[k];
      }
      if (lab[c] >= (uint32_t)NC) atomicOr(label_err, 1);  // training.py:68-69 (np.eye indexing) raises
      const uint32_t v = vme[c];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __fdividef(p[k], ssum);
        const float g = lab[c] == (uint32_t)k ? 1.f : 0.f;
        if (probs) probs[(size_t)v * NC + k] = p[k];
        st[k] += p[k] * g;
        st[NC + k] += p[k];
        st[2 * NC + k] += g;
        st[3 * NC] += -__logf(fmaxf(p[k], clamp)) * g;
      }
      if (pred) {  // np.argmax of these probabilities: the first maximal class
        int a = 0;
#pragma unroll
        for (int k = 1; k < NC; ++k) a = p[k] > p[a] ? k : a;
        pred[v] = (uint8_t)a;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 3 * NC + 1; ++k) {
    float s = block_sum(st[k], red);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.x * (3 * NC + 1) + k] = s;
  }
}

// Head backward for C = 16 / 32 on rows whose width is a multiple of 32 (every U-Net level
// here): a warp owns 32 consecutive voxels of one row, a team of TPV = C/8 lanes owns TPV of
// them (voxel u*(32/TPV) + team, u < TPV), each lane one 8-channel group of all TPV.  The
// per-voxel softmax + loss gradient runs ONCE per voxel: the logit partials are
// reduce-scattered over the team (lane cg ends with voxel cg's logits), lane cg computes that
// voxel's dL/dlogits, and the team all-gathers them.  k_head_bwd_grp computed the softmax on
// every lane of the group (TPV x the per-voxel scalar work) and decomposed every voxel index:
// 800 thread instructions per voxel, issue-bound at ~0.3 of HBM.  Same partial layout.
template <typename T, int C, int NC>
__global__ void __launch_bounds__(kHeadThreads, 2) k_head_bwd_team(
    const T* __restrict__ y, Slab sy, const float* __restrict__ W, const float* __restrict__ bias,
    const uint8_t* __restrict__ labels, const float* __restrict__ stats, T* __restrict__ g, Slab sg,
    float* __restrict__ wpart, int B, float w_dice, float w_ce, float total, int dice_mask, float clamp,
    int relu_mask, const float* __restrict__ dprobs) {
  static_assert(C == 16 || C == 32, "team kernel: C = 16 or 32");
  pdl_wait();
  constexpr int TPV = C / 8;          // lanes per team = voxels per team
  constexpr int TW = 32 / TPV;        // teams per warp
  constexpr int NACC = 8 * NC + NC;   // this lane's channel group's weight grads + bias grads
  constexpr int NWARP = kHeadThreads / 32;
  // 32-voxel chunks per warp iteration, all loads issued first: 4 x 16 B per lane in flight
  // (2 x 16 B at C = 16 with one chunk held the kernel to ~2.2 TB/s, latency-bound)
  constexpr int CH = TPV == 2 ? 2 : 1;
  __shared__ float sW[C * NC], sb[NC], coef[3 * NC];
  __shared__ float red[NWARP][TPV][NACC];
  for (int i = threadIdx.x; i < C * NC; i += blockDim.x) sW[i] = W[i];
  if (threadIdx.x < NC) sb[threadIdx.x] = bias[threadIdx.x];
  if (threadIdx.x == 0) {
    const int nfg = __popc(dice_mask);
    for (int k = 0; k < NC; ++k) {  // training.py:119-124
      const float nk = stats ? 2.f * stats[k] + 1e-6f : 1.f;
      const float dk = stats ? stats[NC + k] + stats[2 * NC + k] + 1e-6f : 1.f;
      const bool on = (dice_mask >> k) & 1;
      coef[3 * k + 0] = on ? (-w_dice / (float)nfg) / dk : 0.f;
      coef[3 * k + 1] = on ? nk / dk : 0.f;
      coef[3 * k + 2] = on ? 1.f : 0.f;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane % TPV, team = lane / TPV, base = lane - cg;
  const float* wr = sW + cg * 8 * NC;  // shared: TPV distinct banks per warp, no conflicts
  const float ce_scale = -w_ce / total;
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.f;
  const uint32_t nchunk = (uint32_t)B * sy.D * sy.H * (sy.W / 32);
  const uint32_t wstride = gridDim.x * NWARP;
  for (uint32_t ch0 = blockIdx.x * NWARP + warp; ch0 < nchunk; ch0 += CH * wstride) {
    float yv[CH][TPV][8];
    int64_t go[CH];
    uint32_t vme[CH];
    int lab[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t ch = min(ch0 + c * wstride, nchunk - 1);  // a clamped duplicate is not stored
      const uint32_t v0 = ch * 32;
      int b, d, h, w0;
      decompose(v0, sy, b, d, h, w0);
      const int64_t yo = sy.at(b, cg, d, h, w0 + team);
      go[c] = sg.at(b, cg, d, h, w0 + team);
#pragma unroll
      for (int u = 0; u < TPV; ++u) V8<T>::ld(y + yo + (int64_t)u * TW * 8, yv[c][u]);
      vme[c] = v0 + cg * TW + team;  // this lane's voxel for the scalar work: u = cg
      lab[c] = labels && !dprobs ? (int)labels[vme[c]] : 255;
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const bool live = ch0 + c * wstride < nchunk;  // warp-uniform
      // logit partials of this lane's 8 channels for all TPV voxels
      float pl[TPV][NC];
#pragma unroll
      for (int u = 0; u < TPV; ++u)
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          float t = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) t = fmaf(yv[c][u][j], wr[j * NC + k], t);
          pl[u][k] = t;
        }
      // reduce-scatter over the team: lane cg keeps the sum for voxel u = cg
      float lg[NC];
      team_reduce_scatter<TPV, NC>(pl, cg, lg);
#pragma unroll
      for (int k = 0; k < NC; ++k) lg[k] += sb[k];
      float m = lg[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) m = fmaxf(m, lg[k]);
      float p[NC], ssum = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __expf(lg[k] - m);
        ssum += p[k];
      }
      float gp[NC], dot = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        p[k] = __fdividef(p[k], ssum);
        const float gk = lab[c] == k ? 1.f : 0.f;
        float r = coef[3 * k + 2] != 0.f ? coef[3 * k] * (2.f * gk - coef[3 * k + 1]) : 0.f;
        // one-hot g: only the label's class has a cross-entropy term (training.py:125-126)
        r += (lab[c] == k && p[k] >= clamp) ? ce_scale * __frcp_rn(p[k]) : 0.f;
        if (dprobs) r = dprobs[(size_t)vme[c] * NC + k];  // external dL/dp
        gp[k] = r;
        dot += r * p[k];
      }
      float gl[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        gl[k] = live ? p[k] * (gp[k] - dot) : 0.f;  // ops.py:197-199
        acc[8 * NC + k] += gl[k];                   // bias: every voxel once (its own lane)
      }
      // all-gather the team's dL/dlogits and finish every voxel's 8 channels of this lane
#pragma unroll
      for (int u = 0; u < TPV; ++u) {
        float gu[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) gu[k] = __shfl_sync(0xffffffffu, gl[k], base + u);
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float sacc = 0.f;
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            sacc = fmaf(wr[j * NC + k], gu[k], sacc);
            acc[j * NC + k] = fmaf(yv[c][u][j], gu[k], acc[j * NC + k]);
          }
          o[j] = (relu_mask && !(yv[c][u][j] > 0.f)) ? 0.f : sacc;
        }
        if (live) V8<T>::st(g + go[c] + (int64_t)u * TW * 8, o);
      }
    }
  }
  // reduce over the lanes of this warp holding the same group, then over warps (fixed order);
  // bias sums live on every lane (one voxel each) and are reduced over all 32 lanes
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    float t = acc[i];
    if (i >= 8 * NC) {
#pragma unroll
      for (int o = 1; o < TPV; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
#pragma unroll
    for (int o = TPV; o < 32; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane < TPV) red[warp][lane][i] = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C * NC + NC; i += blockDim.x) {
    float t = 0.f;
    if (i < C * NC) {
      const int c = i / NC, k = i % NC;
      for (int wq = 0; wq < NWARP; ++wq) t += red[wq][c / 8][(c % 8) * NC + k];
    } else {
      for (int wq = 0; wq < NWARP; ++wq) t += red[wq][0][8 * NC + (i - C * NC)];
    }
    wpart[(int64_t)blockIdx.x * (C * NC + NC) + i] = t;
  }
}

// one block per column: thread t sums rows t, t+256, ... (a few independent loads), then a
// fixed shared-memory tree (deterministic).  One warp per column looped ~20 dependent L2
// round trips over the 592 partial rows (7 us per call).
__global__ void __launch_bounds__(256) k_reduce_rows(const float* __restrict__ part, int rows, int width,
                                                     float* __restrict__ out) {
  __shared__ float red[256];
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x;
  float s = 0.f;
  for (int r = threadIdx.x; r < rows; r += 256) s += part[(int64_t)r * width + j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = red[0];
}

// ------------------------------------------------------------------ SGD (training.py:202-219)
// Grid-stride over the whole flat parameter buffer (balanced across layers of very different
// sizes; a per-layer grid.y left the deep layers' blocks looping alone), the layer of an element
// found by binary search over the offsets cached in shared memory.
constexpr int kSgdMaxLayers = 512;
__device__ __forceinline__ int sgd_layer(const int64_t* soff, int nl, int64_t i) {
  int lo = 0, hi = nl - 1;  // last layer with off[l] <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (soff[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void k_sgd_check(const float* __restrict__ g, const int64_t* __restrict__ off, int nl,
                            int* __restrict__ flags) {
  __shared__ int64_t soff[kSgdMaxLayers + 1];
  pdl_wait();
  for (int i = threadIdx.x; i <= nl; i += blockDim.x) soff[i] = off[i];
  __syncthreads();
  const int64_t a = soff[0], n = soff[nl];
  // 4 elements per thread (16-byte loads from a 16-byte aligned base); the layer lookup only
  // for the rare non-finite element
  for (int64_t i = (a & ~3LL) + 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i < n;
       i += 4 * (int64_t)gridDim.x * blockDim.x) {
    if (i >= a && i + 4 <= n && (reinterpret_cast<uintptr_t>(g + i) & 15) == 0) {
      const float4 v = *reinterpret_cast<const float4*>(g + i);
      if (isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w)) continue;
    }
    for (int64_t j = i; j < i + 4 && j < n; ++j)
      if (j >= a && !isfinite(g[j])) atomicOr(&flags[sgd_layer(soff, nl, j)], 1);  // rare
  }
}

__global__ void k_sgd_apply(float* __restrict__ p, float* __restrict__ v, const float* __restrict__ g,
                            const int64_t* __restrict__ off, int nl, const int* __restrict__ flags, float lr,
                            float mu) {
  __shared__ int64_t soff[kSgdMaxLayers + 1];
  __shared__ int sflag[kSgdMaxLayers];
  pdl_wait();
  for (int i = threadIdx.x; i <= nl; i += blockDim.x) {
    soff[i] = off[i];
    if (i < nl) sflag[i] = flags[i];
  }
  __syncthreads();
  const int64_t a = soff[0], n = soff[nl];
  // numpy fp32 order: v *= mu; v += g; p -= lr * v   (no FMA contraction)
  auto upd = [&](float& pp, float& vv, float gg) {
    vv = __fadd_rn(__fmul_rn(vv, mu), gg);
    pp = __fsub_rn(pp, __fmul_rn(lr, vv));
  };
  // 4 elements per thread: one layer lookup when all four are in the same layer
  for (int64_t i = (a & ~3LL) + 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i < n;
       i += 4 * (int64_t)gridDim.x * blockDim.x) {
    const bool vec = i >= a && i + 4 <= n && ((reinterpret_cast<uintptr_t>(p + i) | reinterpret_cast<uintptr_t>(v + i) |
                                               reinterpret_cast<uintptr_t>(g + i)) & 15) == 0;
    const int l0 = sgd_layer(soff, nl, i >= a ? i : a);
    if (vec && (l0 + 1 >= nl + 1 || soff[l0 + 1] >= i + 4)) {  // all four in layer l0
      if (sflag[l0]) continue;
      float4 pp = *reinterpret_cast<float4*>(p + i), vv = *reinterpret_cast<float4*>(v + i);
      const float4 gg = *reinterpret_cast<const float4*>(g + i);
      upd(pp.x, vv.x, gg.x);
      upd(pp.y, vv.y, gg.y);
      upd(pp.z, vv.z, gg.z);
      upd(pp.w, vv.w, gg.w);
      *reinterpret_cast<float4*>(v + i) = vv;
      *reinterpret_cast<float4*>(p + i) = pp;
      continue;
    }
    for (int64_t j = i; j < i + 4 && j < n; ++j) {
      if (j < a || sflag[sgd_layer(soff, nl, j)]) continue;
      float pp = p[j], vv = v[j];
      upd(pp, vv, g[j]);
      v[j] = vv;
      p[j] = pp;
    }
  }
}

}  // namespace vm

using namespace vm;

#define SLAB(bs, C, D, H, W) make_slab((bs) ? (bs) : default_bstride((C), (D), (H), (W), 1), ((C) + 7) / 8, (D), (H), (W), 1)

#define DISPATCH_T(dtype, NAME, ...)                                  \
  do {                                                                \
    if ((dtype) == VM_BF16) {                                         \
      using T = __nv_bfloat16;                                        \
      __VA_ARGS__;                                                    \
    } else if ((dtype) == VM_F32) {                                   \
      using T = float;                                                \
      __VA_ARGS__;                                                    \
    } else {                                                          \
      VM_REQUIRE(false, VM_E_DTYPE, "%s: dtype %d", NAME, (dtype));   \
    }                                                                 \
  } while (0)

extern "C" int vm_maxpool2_fwd(int dtype, const void* x, int64_t x_bstride, void* y,
                               int64_t y_bstride, int B, int C, int D, int H, int W, void* stream) {
  VM_REQUIRE(x && y, VM_E_ARG, "vm_maxpool2_fwd: null pointer");
  VM_REQUIRE(D % 2 == 0 && H % 2 == 0 && W % 2 == 0, VM_E_SHAPE,
             "maxpool2 needs even local extents, got (%d, %d, %d)", D, H, W);
  Slab gx = SLAB(x_bstride, C, D, H, W), gy = SLAB(y_bstride, C, D / 2, H / 2, W / 2);
  int64_t work = (int64_t)B * (D / 2) * (H / 2) * (W / 2) * gy.CG;
  VM_REQUIRE(work < (1LL << 32), VM_E_SHAPE, "index space %lld exceeds 2^32", (long long)work);
  DISPATCH_T(dtype, "vm_maxpool2_fwd",
             launch_pdl(k_maxpool_fwd<T>, grid_for(work, 256), 256, 0, as_stream(stream),
                 (const T*)x, gx, (T*)y, gy, B));
  return launch_status("vm_maxpool2_fwd");
}

extern "C" int vm_maxpool2_bwd(int dtype, const void* x, int64_t x_bstride, const void* gout,
                               int64_t gout_bstride, const void* add, int64_t add_bstride,
                               void* gin, int64_t gin_bstride, int B, int C, int D, int H, int W,
                               int relu_mask, void* stream) {
  VM_REQUIRE(x && gout && gin, VM_E_ARG, "vm_maxpool2_bwd: null pointer");
  VM_REQUIRE(D % 2 == 0 && H % 2 == 0 && W % 2 == 0, VM_E_SHAPE, "maxpool2_bwd: odd extents");
  Slab gx = SLAB(x_bstride, C, D, H, W), go = SLAB(gout_bstride, C, D / 2, H / 2, W / 2);
  Slab ga = SLAB(add_bstride, C, D, H, W), gi = SLAB(gin_bstride, C, D, H, W);
  int64_t work = (int64_t)B * (D / 2) * (H / 2) * (W / 2) * go.CG;
  VM_REQUIRE(work < (1LL << 32), VM_E_SHAPE, "index space %lld exceeds 2^32", (long long)work);
  DISPATCH_T(dtype, "vm_maxpool2_bwd",
             launch_pdl(k_maxpool_bwd<T>, grid_for(work, 256), 256, 0, as_stream(stream),
                 (const T*)x, gx, (const T*)gout, go, (const T*)add, ga, (T*)gin, gi, B, relu_mask));
  return launch_status("vm_maxpool2_bwd");
}

extern "C" int vm_upsample2_fwd(int dtype, const void* x, int64_t x_bstride, void* y,
                                int64_t y_bstride, int B, int C, int D, int H, int W, void* stream) {
  VM_REQUIRE(x && y, VM_E_ARG, "vm_upsample2_fwd: null pointer");
  Slab gx = SLAB(x_bstride, C, D, H, W), gy = SLAB(y_bstride, C, 2 * D, 2 * H, 2 * W);
  int64_t work = (int64_t)B * D * H * W * gx.CG * 2;  // (input vector, output w parity)
  VM_REQUIRE(work * 4 < (1LL << 32), VM_E_SHAPE, "index space %lld exceeds 2^32", (long long)work * 4);
  DISPATCH_T(dtype, "vm_upsample2_fwd",
             launch_pdl(k_upsample_fwd<T>, grid_for(work, 256), 256, 0, as_stream(stream),
                 (const T*)x, gx, (T*)y, gy, B));
  return launch_status("vm_upsample2_fwd");
}

extern "C" int vm_upsample2_bwd(int dtype, const void* gy, int64_t gy_bstride, const void* mask,
                                int64_t mask_bstride, void* gx, int64_t gx_bstride, int B, int C,
                                int D, int H, int W, void* stream) {
  VM_REQUIRE(gy && gx, VM_E_ARG, "vm_upsample2_bwd: null pointer");
  Slab sgy = SLAB(gy_bstride, C, 2 * D, 2 * H, 2 * W), sgx = SLAB(gx_bstride, C, D, H, W);
  Slab sm = SLAB(mask_bstride, C, D, H, W);
  int64_t work = (int64_t)B * D * H * W * sgx.CG;
  VM_REQUIRE(work < (1LL << 32), VM_E_SHAPE, "index space %lld exceeds 2^32", (long long)work);
  DISPATCH_T(dtype, "vm_upsample2_bwd",
             launch_pdl(k_upsample_bwd<T>, grid_for(work, 256), 256, 0, as_stream(stream),
                 (const T*)gy, sgy, (const T*)mask, sm, (T*)gx, sgx, B));
  return launch_status("vm_upsample2_bwd");
}

extern "C" int vm_relu_mask(int dtype, const void* g, int64_t g_bstride, const void* mask,
                            int64_t mask_bstride, void* out, int64_t out_bstride, int B, int C,
                            int D, int H, int W, void* stream) {
  VM_REQUIRE(g && mask && out, VM_E_ARG, "vm_relu_mask: null pointer");
  Slab sg = SLAB(g_bstride, C, D, H, W), sm = SLAB(mask_bstride, C, D, H, W);
  Slab so = SLAB(out_bstride, C, D, H, W);
  int64_t work = (int64_t)B * D * H * W * sg.CG;
  VM_REQUIRE(work < (1LL << 32), VM_E_SHAPE, "index space %lld exceeds 2^32", (long long)work);
  DISPATCH_T(dtype, "vm_relu_mask",
             k_relu_mask<T><<<grid_for(work, 256), 256, 0, as_stream(stream)>>>(
                 (const T*)g, sg, (const T*)mask, sm, (T*)out, so, B));
  return launch_status("vm_relu_mask");
}

extern "C" int vm_head_partials_count(int B, int D, int H, int W) {
  int64_t nvox = (int64_t)B * D * H * W;
  int64_t blocks = (nvox + kHeadThreads - 1) / kHeadThreads;
  int cap = 148 * 2;  // one wave of 2 resident 256-thread blocks per SM (register-limited)
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

static int g_head_team_off = 0;  // vm_debug_set_head_team (A/B against the per-voxel / per-group kernels)
extern "C" void vm_debug_set_head_team(int on) { g_head_team_off = !on; }

extern "C" int vm_head_fwd(int dtype, const void* y, int64_t y_bstride, const float* w,
                           const float* b, const uint8_t* labels, int* label_err, float* probs,
                           uint8_t* pred, float* partials, int B, int C, int ncls, int D, int H, int W, float clamp, void* stream) {
  VM_REQUIRE(y && w && b && labels && label_err && partials, VM_E_ARG, "vm_head_fwd: null pointer");
  VM_REQUIRE(ncls > 0 && ncls <= kMaxCls, VM_E_UNSUPPORTED, "vm_head_fwd: ncls %d > %d", ncls, kMaxCls);
  VM_REQUIRE((int64_t)B * D * H * W < (1LL << 32), VM_E_SHAPE, "vm_head_fwd: voxel count exceeds 2^32");
  Slab sy = SLAB(y_bstride, C, D, H, W);
  int grid = vm_head_partials_count(B, D, H, W);
  size_t sh = (C * ncls + ncls + 32) * sizeof(float);
  if (dtype == VM_BF16) {  // fixed-width kernels: C in {8, 16, 32, 64}, 2..4 classes
    using T = __nv_bfloat16;
    auto st = as_stream(stream);
    // (C = 16: the per-voxel kernel with two voxels in flight is faster, 22 vs 25 us at 128^3)
    if (C == 32 && W % 32 == 0 && !g_head_team_off) {
#define HT_CASE(CC, NN)                                                                                  \
  case NN * 1000 + CC:                                                                                   \
    launch_pdl(k_head_fwd_team<T, CC, NN>, grid, kHeadThreads, 0, st, (const T*)y, sy, w, b, labels,         \
               label_err, probs, pred, partials, B, clamp);                                                         \
    return launch_status("vm_head_fwd");
      switch (ncls * 1000 + C) {
        HT_CASE(32, 2) HT_CASE(32, 3) HT_CASE(32, 4)
        default:
          break;
      }
#undef HT_CASE
    }
#define HF_CASE(CC, NN)                                                                               \
  case NN * 1000 + CC:                                                                                \
    launch_pdl(k_head_fwd_fixed<T, CC, NN>, grid, kHeadThreads, 0, st, (const T*)y, sy, w, b, labels, \
               label_err, probs, pred, partials, B, clamp);                                                            \
    return launch_status("vm_head_fwd");
#define HF_ROW(NN) HF_CASE(8, NN) HF_CASE(16, NN) HF_CASE(32, NN) HF_CASE(64, NN)
    switch (ncls * 1000 + C) {
      HF_ROW(2)
      HF_ROW(3)
      HF_ROW(4)
      default:
        break;
    }
#undef HF_ROW
#undef HF_CASE
  }
  DISPATCH_T(dtype, "vm_head_fwd",
             k_head_fwd<T><<<grid, kHeadThreads, sh, as_stream(stream)>>>(
                 (const T*)y, sy, w, b, labels, label_err, probs, pred, partials, B, C, ncls, clamp));
  return launch_status("vm_head_fwd");
}

// Hard-Dice counts of a prediction (training.py:166-194): per class k, |pred==k & gt==k|,
// |pred==k|, |gt==k| as exact 64-bit integers (integer atomics: order-independent, so the
// result is deterministic).  16 voxels per thread per iteration (one 16-byte load of each).
__global__ void k_label_counts(const uint8_t* __restrict__ pred, const uint8_t* __restrict__ gt, int64_t n,
                               int ncls, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int sc[3 * kMaxCls];
  for (int i = threadIdx.x; i < 3 * ncls; i += blockDim.x) sc[i] = 0u;
  __syncthreads();
  unsigned int loc[3 * kMaxCls];
#pragma unroll
  for (int i = 0; i < 3 * kMaxCls; ++i) loc[i] = 0u;
  const int64_t n16 = n / 16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto tally = [&](uint32_t p, uint32_t g) {
#pragma unroll
    for (int k = 0; k < kMaxCls; ++k) {
      loc[k] += (p == (uint32_t)k) & (g == (uint32_t)k);
      loc[kMaxCls + k] += p == (uint32_t)k;
      loc[2 * kMaxCls + k] += g == (uint32_t)k;
    }
  };
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n16; q += stride) {
    const uint4 pv = reinterpret_cast<const uint4*>(pred)[q];
    const uint4 gv = reinterpret_cast<const uint4*>(gt)[q];
    const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) tally((pw[j / 4] >> (8 * (j % 4))) & 0xFFu, (gw[j / 4] >> (8 * (j % 4))) & 0xFFu);
  }
  for (int64_t i = n16 * 16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) tally(pred[i], gt[i]);
  for (int k = 0; k < ncls; ++k) {
    atomicAdd(&sc[k], loc[k]);
    atomicAdd(&sc[ncls + k], loc[kMaxCls + k]);
    atomicAdd(&sc[2 * ncls + k], loc[2 * kMaxCls + k]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * ncls; i += blockDim.x) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

extern "C" int vm_label_counts(const uint8_t* pred, const uint8_t* gt, int64_t n, int ncls,
                               unsigned long long* counts, void* stream) {
  VM_REQUIRE(pred && gt && counts && n >= 0 && ncls > 0 && ncls <= kMaxCls, VM_E_ARG, "vm_label_counts: bad argument");
  VM_REQUIRE(((reinterpret_cast<uintptr_t>(pred) | reinterpret_cast<uintptr_t>(gt)) & 15) == 0, VM_E_ARG,
             "vm_label_counts: pred / gt must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 3 * ncls, st);
  if (n == 0) return launch_status("vm_label_counts");
  const int64_t blocks = (n / 16 + 255) / 256;
  k_label_counts<<<(int)(blocks < 1 ? 1 : (blocks > 2 * 148 ? 2 * 148 : blocks)), 256, 0, st>>>(pred, gt, n, ncls,
                                                                                                counts);
  return launch_status("vm_label_counts");
}

extern "C" int vm_reduce_rows(const float* partials, int rows, int width, float* out, void* stream) {
  VM_REQUIRE(partials && out && rows > 0 && width > 0, VM_E_ARG, "vm_reduce_rows: bad argument");
  launch_pdl(k_reduce_rows, width, 256, 0, as_stream(stream), partials, rows, width, out);
  return launch_status("vm_reduce_rows");
}

static int head_bwd(int dtype, const void* y, int64_t y_bstride, const float* w, const float* b,
                    const uint8_t* labels, const float* stats, void* g, int64_t g_bstride, float* wpartials, int B,
                    int C, int ncls, int D, int H, int W, float w_dice, float w_ce, float total_voxels,
                    int dice_mask, float clamp, int relu_mask, const float* dprobs, void* stream);

extern "C" int vm_head_bwd(int dtype, const void* y, int64_t y_bstride, const float* w,
                           const float* b, const uint8_t* labels, const float* stats, void* g,
                           int64_t g_bstride, float* wpartials, int B, int C, int ncls, int D,
                           int H, int W, float w_dice, float w_ce, float total_voxels,
                           int dice_mask, float clamp, int relu_mask, void* stream) {
  VM_REQUIRE(labels && stats, VM_E_ARG, "vm_head_bwd: null pointer");
  return head_bwd(dtype, y, y_bstride, w, b, labels, stats, g, g_bstride, wpartials, B, C, ncls, D, H, W, w_dice,
                  w_ce, total_voxels, dice_mask, clamp, relu_mask, nullptr, stream);
}

// Head backward from a given dL/dprobs [B][D][H][W][ncls] (f32): softmax backward + head dgrad
// (masked) + head-weight partials, for the worker-level API (unet.run_backward_local fed by
// training.loss_grad_local, unet.py:376-442).
extern "C" int vm_head_bwd_dprobs(int dtype, const void* y, int64_t y_bstride, const float* w, const float* b,
                                  const float* dprobs, void* g, int64_t g_bstride, float* wpartials, int B, int C,
                                  int ncls, int D, int H, int W, int relu_mask, void* stream) {
  VM_REQUIRE(dprobs, VM_E_ARG, "vm_head_bwd_dprobs: null dprobs");
  return head_bwd(dtype, y, y_bstride, w, b, nullptr, nullptr, g, g_bstride, wpartials, B, C, ncls, D, H, W, 0.f,
                  0.f, 1.f, 0, 0.f, relu_mask, dprobs, stream);
}

static int head_bwd(int dtype, const void* y, int64_t y_bstride, const float* w, const float* b,
                    const uint8_t* labels, const float* stats, void* g, int64_t g_bstride, float* wpartials, int B,
                    int C, int ncls, int D, int H, int W, float w_dice, float w_ce, float total_voxels,
                    int dice_mask, float clamp, int relu_mask, const float* dprobs, void* stream) {
  VM_REQUIRE(y && w && b && g && wpartials, VM_E_ARG, "vm_head_bwd: null pointer");
  VM_REQUIRE(ncls > 0 && ncls <= kMaxCls, VM_E_UNSUPPORTED, "vm_head_bwd: ncls %d", ncls);
  VM_REQUIRE((int64_t)B * D * H * W < (1LL << 32), VM_E_SHAPE, "vm_head_bwd: voxel count exceeds 2^32");
  Slab sy = SLAB(y_bstride, C, D, H, W), sg = SLAB(g_bstride, C, D, H, W);
  int grid = vm_head_partials_count(B, D, H, W);
  size_t sh = (C * ncls + ncls + 32 + 3 * kMaxCls) * sizeof(float);
  if (dtype == VM_BF16) {  // fixed-width kernels: C in {8, 16, 32, 64, 128}, 2..4 classes (the
    using T = __nv_bfloat16;  // generic one-thread-per-voxel kernel took 38.7 ms at 256^3, C = 64)
    auto st = as_stream(stream);
    if ((C == 16 || C == 32) && W % 32 == 0 && !g_head_team_off) {
#define HT_CASE(CC, NN)                                                                                  \
  case NN * 1000 + CC:                                                                                   \
    launch_pdl(k_head_bwd_team<T, CC, NN>, grid, kHeadThreads, 0, st, (const T*)y, sy, w, b, labels, stats,   \
               (T*)g, sg, wpartials, B, w_dice, w_ce, total_voxels, dice_mask, clamp, relu_mask, dprobs);          \
    return launch_status("vm_head_bwd");
      switch (ncls * 1000 + C) {
        HT_CASE(16, 2) HT_CASE(32, 2) HT_CASE(16, 3) HT_CASE(32, 3) HT_CASE(16, 4) HT_CASE(32, 4)
        default:
          break;
      }
#undef HT_CASE
    }
#define HB_CASE(CC, NN)                                                                                  \
  case NN * 1000 + CC:                                                                                   \
    launch_pdl(k_head_bwd_grp<T, CC, NN>, grid, kHeadThreads, 0, st, (const T*)y, sy, w, b, labels, stats, \
               (T*)g, sg, wpartials, B, w_dice, w_ce, total_voxels, dice_mask, clamp, relu_mask, dprobs);          \
    return launch_status("vm_head_bwd");
#define HB_ROW(NN) HB_CASE(8, NN) HB_CASE(16, NN) HB_CASE(32, NN) HB_CASE(64, NN) HB_CASE(128, NN)
    switch (ncls * 1000 + C) {
      HB_ROW(2)
      HB_ROW(3)
      HB_ROW(4)
      default:
        break;
    }
#undef HB_ROW
#undef HB_CASE
  }
  DISPATCH_T(dtype, "vm_head_bwd",
             k_head_bwd<T><<<grid, kHeadThreads, sh, as_stream(stream)>>>(
                 (const T*)y, sy, w, b, labels, stats, (T*)g, sg, wpartials, B, C, ncls, w_dice,
                 w_ce, total_voxels, dice_mask, clamp, relu_mask, dprobs));
  return launch_status("vm_head_bwd");
}

extern "C" int vm_sgd_momentum(float* params, float* moments, const float* grads,
                               const int64_t* offsets, int nlayers, int64_t max_layer_elems,
                               int* flags, float lr, float momentum, void* stream) {
  VM_REQUIRE(params && moments && grads && offsets && flags && nlayers > 0, VM_E_ARG,
             "vm_sgd_momentum: bad argument");
  cudaStream_t st = as_stream(stream);
  VM_REQUIRE(nlayers <= kSgdMaxLayers, VM_E_UNSUPPORTED, "vm_sgd_momentum: %d layers > %d", nlayers, kSgdMaxLayers);
  cudaMemsetAsync(flags, 0, sizeof(int) * nlayers, st);
  const int grid = grid_for(max_layer_elems * nlayers, 256);  // upper bound of the buffer size
  launch_pdl(k_sgd_check, grid, 256, 0, st, grads, offsets, nlayers, flags);
  launch_pdl(k_sgd_apply, grid, 256, 0, st, params, moments, grads, offsets, nlayers, (const int*)flags, lr,
             momentum);
  return launch_status("vm_sgd_momentum", 2);
}
