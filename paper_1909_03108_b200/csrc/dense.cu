// dense.cu — the per-op API's row-major kernels (tensors [..., C] with C innermost): channel
// softmax (ops.py:190-194), channel concat (ops.py:313-323), loss statistics and the per-voxel
// loss gradient (training.py:77-127) over probabilities and one-hot labels.  The train step
// fuses all of these into its head kernels (pointwise.cu); these serve the reference's
// op-level / worker-level API (ops.softmax_channels, ops.concat_channels, training.soft_dice_loss
// / cross_entropy_loss / combined_loss, training.loss_stats_local / loss_grad_local).
// HBM-bound; one thread per row (C <= 8 classes) or a grid-stride copy.
#include "vm_common.cuh"

namespace vm {

constexpr int kDenseMaxC = 64;

template <typename T>
__global__ void k_softmax_rows(const T* __restrict__ x, T* __restrict__ y, int64_t rows, int C) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const T* xr = x + r * C;
    float m = Cvt<T>::to_f(xr[0]);
    for (int c = 1; c < C; ++c) m = fmaxf(m, Cvt<T>::to_f(xr[c]));
    float e[kDenseMaxC], s = 0.f;
    for (int c = 0; c < C; ++c) {
      e[c] = expf(Cvt<T>::to_f(xr[c]) - m);
      s += e[c];
    }
    for (int c = 0; c < C; ++c) y[r * C + c] = Cvt<T>::from_f(e[c] / s);
  }
}

__global__ void k_concat_rows(const uint8_t* __restrict__ a, int64_t ab, const uint8_t* __restrict__ b, int64_t bb,
                              uint8_t* __restrict__ out, int64_t rows) {
  const int64_t ob = ab + bb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ob; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ob, c = i - r * ob;
    out[i] = c < ab ? a[r * ab + c] : b[r * bb + (c - ab)];
  }
}

// Loss statistics per block: [sum p*g (C), sum p (C), sum g (C), sum -log(max(p, clamp))*g],
// accumulated in float64 (more accurate than the reference's probs-dtype sums, training.py:84),
// block partials reduced in fixed order by vm_reduce_rows_f64.
__global__ void k_loss_stats(const float* __restrict__ p, const float* __restrict__ g, int64_t rows, int C,
                             float clamp, double* __restrict__ partials) {
  double st[3 * 8 + 1];
  for (int k = 0; k < 3 * C + 1; ++k) st[k] = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < C; ++k) {
      const double pk = p[r * C + k], gk = g[r * C + k];
      st[k] += pk * gk;
      st[C + k] += pk;
      st[2 * C + k] += gk;
      st[3 * C] += -log(fmax(pk, (double)clamp)) * gk;
    }
  }
  __shared__ double red[8][3 * 8 + 1];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int k = 0; k < 3 * C + 1; ++k) {
    double v = st[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3 * C + 1) {
    double s = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) s += red[w][threadIdx.x];
    partials[(int64_t)blockIdx.x * (3 * C + 1) + threadIdx.x] = s;
  }
}

__global__ void k_reduce_rows_f64(const double* __restrict__ partials, int nrows, int width, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= width) return;
  double s = 0.0;
  for (int i = 0; i < nrows; ++i) s += partials[(int64_t)i * width + k];  // fixed order
  out[k] = s;
}

// dL/dp per voxel (training.py:110-127): soft-Dice over the classes of dice_mask plus the
// clamped cross-entropy term, from the globally reduced statistics.
__global__ void k_loss_grad(const float* __restrict__ p, const float* __restrict__ g, const double* __restrict__ stats,
                            int64_t rows, int C, float w_dice, float w_ce, double total, int dice_mask, float clamp,
                            float* __restrict__ out) {
  const int nfg = __popc(dice_mask);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < C; ++k) {
      const double pk = p[r * C + k], gk = g[r * C + k];
      double v = 0.0;
      if ((dice_mask >> k) & 1) {
        const double nk = 2.0 * stats[k] + 1e-6, dk = stats[C + k] + stats[2 * C + k] + 1e-6;
        v += (-(double)w_dice / nfg) * ((2.0 * gk - nk / dk) / dk);
      }
      if (pk >= clamp) v += (-(double)w_ce / total) * (gk / fmax(pk, (double)clamp));
      out[r * C + k] = (float)v;
    }
  }
}

}  // namespace vm

using namespace vm;

extern "C" int vm_softmax_rows(int dtype, const void* x, void* y, int64_t rows, int C, void* stream) {
  VM_REQUIRE(x && y && rows >= 0 && C > 0 && C <= kDenseMaxC, VM_E_ARG, "vm_softmax_rows: bad argument (C=%d)", C);
  if (rows == 0) return VM_OK;
  const int grid = grid_for(rows, 256);
  if (dtype == VM_F32) k_softmax_rows<float><<<grid, 256, 0, as_stream(stream)>>>((const float*)x, (float*)y, rows, C);
  else if (dtype == VM_BF16)
    k_softmax_rows<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y,
                                                                        rows, C);
  else VM_REQUIRE(false, VM_E_DTYPE, "vm_softmax_rows: dtype %d", dtype);
  return launch_status("vm_softmax_rows");
}

extern "C" int vm_concat_rows(const void* a, int64_t a_row_bytes, const void* b, int64_t b_row_bytes, void* out,
                              int64_t rows, void* stream) {
  VM_REQUIRE(a && b && out && rows >= 0, VM_E_ARG, "vm_concat_rows: bad argument");
  const int64_t total = rows * (a_row_bytes + b_row_bytes);
  if (total == 0) return VM_OK;
  k_concat_rows<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      (const uint8_t*)a, a_row_bytes, (const uint8_t*)b, b_row_bytes, (uint8_t*)out, rows);
  return launch_status("vm_concat_rows");
}

// stats (f64, 3*C+1) of probabilities / one-hot labels [rows, C] (f32); ws: 2*148*(3C+1) doubles
extern "C" int vm_loss_stats(const float* probs, const float* onehot, int64_t rows, int C, float clamp, double* ws,
                             double* stats, void* stream) {
  VM_REQUIRE(probs && onehot && ws && stats && C > 0 && C <= 8, VM_E_ARG, "vm_loss_stats: bad argument");
  int grid = (int)((rows + 255) / 256);
  grid = grid < 1 ? 1 : (grid > 2 * 148 ? 2 * 148 : grid);
  k_loss_stats<<<grid, 256, 0, as_stream(stream)>>>(probs, onehot, rows, C, clamp, ws);
  k_reduce_rows_f64<<<1, 32, 0, as_stream(stream)>>>(ws, grid, 3 * C + 1, stats);
  return launch_status("vm_loss_stats", 2);
}

extern "C" int vm_loss_grad(const float* probs, const float* onehot, const double* stats, int64_t rows, int C,
                            float w_dice, float w_ce, double total, int dice_mask, float clamp, float* out,
                            void* stream) {
  VM_REQUIRE(probs && onehot && stats && out && C > 0 && C <= 8, VM_E_ARG, "vm_loss_grad: bad argument");
  if (rows == 0) return VM_OK;
  k_loss_grad<<<grid_for(rows, 256), 256, 0, as_stream(stream)>>>(probs, onehot, stats, rows, C, w_dice, w_ce, total,
                                                                   dice_mask, clamp, out);
  return launch_status("vm_loss_grad");
}
