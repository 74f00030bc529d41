// augment.cu — tumour remove / synthesise augmentation on the GPU,
// restating voxmesh augment.py:53-151 for device-resident volumes.
//
//   intensity_delta   (augment.py:53-64)   vm_aug_stats: f64 sums over tumour / liver voxels
//   remove_tumor      (augment.py:67-78)   vm_aug_remove: image -= f32(delta), label 2 -> 1
//   synthesize_tumor  (augment.py:89-134)  vm_aug_paint (f64 ellipsoid test, the reference's
//                                          accumulation order), vm_aug_blur_axis (scipy
//                                          correlate1d order, double accumulate, f32 out),
//                                          vm_aug_finish (clip, liver mask, image += d*w,
//                                          labels where w >= threshold)
// The random draws (tumour count, centres, radii) and the Gaussian weights stay on the host
// with numpy, exactly as the reference computes them; vm_aug_count_chunks lets the host find
// the k-th liver voxel (np.argwhere order) without copying the label volume.  All volumes are
// dense C-order [D][H][W] (image f32, labels u8).  HBM-bound elementwise / stencil kernels.
#include "vm_common.cuh"

namespace vm {
namespace {

constexpr int kAugThreads = 256;
constexpr int kAugStatBlocks = 592;  // fixed: the f64 sums are reduced in a fixed order

// per block: [sum(image | tumour), #tumour, sum(image | liver), #liver] over a fixed
// contiguous chunk, thread-strided then tree-reduced (deterministic)
__global__ void __launch_bounds__(kAugThreads) k_aug_stats(const float* __restrict__ img,
                                                           const uint8_t* __restrict__ lab, int64_t n,
                                                           double* __restrict__ part) {
  __shared__ double red[4][kAugThreads];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double st = 0.0, ct = 0.0, sl = 0.0, cl = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint8_t l = lab[i];
    const double v = (double)img[i];
    if (l == 2) {
      st += v;
      ct += 1.0;
    } else if (l == 1) {
      sl += v;
      cl += 1.0;
    }
  }
  red[0][threadIdx.x] = st;
  red[1][threadIdx.x] = ct;
  red[2][threadIdx.x] = sl;
  red[3][threadIdx.x] = cl;
  __syncthreads();
  for (int s = kAugThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int k = 0; k < 4; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void k_aug_stats_final(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[b * 4 + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// augment.py:74-77: image[tumour] -= f32(delta); labels[tumour] = 1
__global__ void k_aug_remove(float* __restrict__ img, uint8_t* __restrict__ lab, int64_t n, float delta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (lab[i] == 2) {
      img[i] = __fsub_rn(img[i], delta);
      lab[i] = 1;
    }
  }
}

// number of voxels with label == value in each chunk of `chunk` consecutive voxels
__global__ void k_aug_count_chunks(const uint8_t* __restrict__ lab, int64_t n, int chunk, int value,
                                   int* __restrict__ counts) {
  __shared__ int red[kAugThreads];
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  int c = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) c += lab[i] == value;
  red[threadIdx.x] = c;
  __syncthreads();
  for (int s = kAugThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[blockIdx.x] = red[0];
}

// mask[v] = 1 where v is liver and inside any ellipsoid: acc = ((g0-c0)/r0)^2, then
// + ((g1-c1)/r1)^2, then + ((g2-c2)/r2)^2 in float64 (augment.py:81-86), acc <= 1
__global__ void k_aug_paint(const uint8_t* __restrict__ lab, int D, int H, int W, const int64_t* __restrict__ centers,
                            const double* __restrict__ radii, int ntum, float* __restrict__ mask) {
  const int64_t n = (int64_t)D * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i / ((int64_t)H * W)), y = (int)((i / W) % H), z = (int)(i % W);
    bool in = false;
    for (int t = 0; t < ntum && !in; ++t) {
      const double a0 = __ddiv_rn((double)(x - centers[3 * t + 0]), radii[3 * t + 0]);
      const double a1 = __ddiv_rn((double)(y - centers[3 * t + 1]), radii[3 * t + 1]);
      const double a2 = __ddiv_rn((double)(z - centers[3 * t + 2]), radii[3 * t + 2]);
      double acc = __dadd_rn(0.0, __dmul_rn(a0, a0));
      acc = __dadd_rn(acc, __dmul_rn(a1, a1));
      acc = __dadd_rn(acc, __dmul_rn(a2, a2));
      in = acc <= 1.0;
    }
    mask[i] = (in && lab[i] == 1) ? 1.f : 0.f;
  }
}

// One scipy.ndimage.correlate1d pass (mode "constant", cval 0) with a symmetric kernel of
// radius r along `axis` of a [D][H][W] f32 volume: in double, out = x[0]*w0, then
// out += (x[-j] + x[+j]) * wj for j = r .. 1 (ni_filters.c NI_Correlate1D, symmetric branch),
// rounded to f32.  No FMA contraction, like the reference build.
__global__ void k_aug_blur_axis(const float* __restrict__ in, float* __restrict__ out, int D, int H, int W,
                                int axis, const double* __restrict__ w, int r) {
  const int64_t n = (int64_t)D * H * W;
  const int64_t stride = axis == 0 ? (int64_t)H * W : axis == 1 ? (int64_t)W : 1;
  const int len = axis == 0 ? D : axis == 1 ? H : W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int pos = (int)((i / stride) % len);
    double acc = __dmul_rn((double)in[i], w[0]);
    for (int j = r; j >= 1; --j) {
      const double left = pos - j >= 0 ? (double)in[i - j * stride] : 0.0;
      const double right = pos + j < len ? (double)in[i + j * stride] : 0.0;
      acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(left, right), w[j]));
    }
    out[i] = __double2float_rn(acc);
  }
}

// augment.py:123-133: w = clip(blur, 0, 1) * liver; image += f32(delta) * w;
// labels = 2 where w >= threshold and liver
__global__ void k_aug_finish(float* __restrict__ img, uint8_t* __restrict__ lab, const float* __restrict__ wv,
                             int64_t n, float delta, float thr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool liver = lab[i] == 1;
    float w = fminf(fmaxf(wv[i], 0.f), 1.f);
    w = __fmul_rn(w, liver ? 1.f : 0.f);
    img[i] = __fadd_rn(img[i], __fmul_rn(delta, w));
    if (liver && w >= thr) lab[i] = 2;
  }
}

}  // namespace
}  // namespace vm

using namespace vm;

extern "C" size_t vm_aug_stats_ws_bytes(void) { return (size_t)kAugStatBlocks * 4 * sizeof(double); }

// out[4] = {sum(image | label 2), #label 2, sum(image | label 1), #label 1} in float64
extern "C" int vm_aug_stats(const float* image, const uint8_t* labels, int64_t n, double* ws, double* out,
                            void* stream) {
  VM_REQUIRE(image && labels && ws && out && n > 0, VM_E_ARG, "vm_aug_stats: bad argument");
  cudaStream_t st = as_stream(stream);
  k_aug_stats<<<kAugStatBlocks, kAugThreads, 0, st>>>(image, labels, n, ws);
  k_aug_stats_final<<<1, 32, 0, st>>>(ws, kAugStatBlocks, out);
  return launch_status("vm_aug_stats", 2);
}

extern "C" int vm_aug_remove(float* image, uint8_t* labels, int64_t n, float delta, void* stream) {
  VM_REQUIRE(image && labels && n > 0, VM_E_ARG, "vm_aug_remove: bad argument");
  k_aug_remove<<<grid_for(n, kAugThreads), kAugThreads, 0, as_stream(stream)>>>(image, labels, n, delta);
  return launch_status("vm_aug_remove");
}

extern "C" int vm_aug_count_chunks(const uint8_t* labels, int64_t n, int chunk, int value, int* counts,
                                   void* stream) {
  VM_REQUIRE(labels && counts && n > 0 && chunk > 0, VM_E_ARG, "vm_aug_count_chunks: bad argument");
  const int64_t nch = (n + chunk - 1) / chunk;
  VM_REQUIRE(nch < (1LL << 31), VM_E_SHAPE, "vm_aug_count_chunks: too many chunks");
  k_aug_count_chunks<<<(unsigned)nch, kAugThreads, 0, as_stream(stream)>>>(labels, n, chunk, value, counts);
  return launch_status("vm_aug_count_chunks");
}

extern "C" int vm_aug_paint(const uint8_t* labels, int D, int H, int W, const int64_t* centers,
                            const double* radii, int ntumours, float* mask, void* stream) {
  VM_REQUIRE(labels && centers && radii && mask && ntumours > 0, VM_E_ARG, "vm_aug_paint: bad argument");
  const int64_t n = (int64_t)D * H * W;
  k_aug_paint<<<grid_for(n, kAugThreads), kAugThreads, 0, as_stream(stream)>>>(labels, D, H, W, centers, radii,
                                                                               ntumours, mask);
  return launch_status("vm_aug_paint");
}

// w[0..r]: the centre weight then j = 1..r (symmetric kernel, host-computed like scipy)
extern "C" int vm_aug_blur_axis(const float* in, float* out, int D, int H, int W, int axis, const double* w, int r,
                                void* stream) {
  VM_REQUIRE(in && out && w && in != out && axis >= 0 && axis < 3 && r >= 0, VM_E_ARG,
             "vm_aug_blur_axis: bad argument");
  const int64_t n = (int64_t)D * H * W;
  k_aug_blur_axis<<<grid_for(n, kAugThreads), kAugThreads, 0, as_stream(stream)>>>(in, out, D, H, W, axis, w, r);
  return launch_status("vm_aug_blur_axis");
}

extern "C" int vm_aug_finish(float* image, uint8_t* labels, const float* w, int64_t n, float delta, float threshold,
                             void* stream) {
  VM_REQUIRE(image && labels && w && n > 0, VM_E_ARG, "vm_aug_finish: bad argument");
  k_aug_finish<<<grid_for(n, kAugThreads), kAugThreads, 0, as_stream(stream)>>>(image, labels, w, n, delta,
                                                                                threshold);
  return launch_status("vm_aug_finish");
}
