// probe_tcgen05.cu — de-risks the conv3d design on a real B200 before the kernels
// are written: (1) row-shifted SWIZZLE_NONE K-major A descriptors, (2) LBO used
// as a "tap distance", (3) MN-major operands, (4) TMA 2-D/3-D boxes into the
// channel-blocked [cg][rows][8] layout, (5) tcgen05.mma SS throughput vs N.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe probe_tcgen05.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

using bf16 = __nv_bfloat16;

// Generic single-MMA test: A, B images are copied verbatim into smem (offsets
// given in bytes), one MMA with the given descriptors, D read back.
struct MmaCase {
  uint32_t a_off, a_lbo, a_sbo;
  uint32_t b_off, b_lbo, b_sbo;
  int M, N;
  int a_mn, b_mn;
};

__global__ void k_single_mma(const uint8_t* img, int img_bytes, MmaCase c, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < img_bytes; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = *reinterpret_cast<const int4*>(img + i);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    vm::mbar_init(&bar, 1);
    vm::fence_barrier_init();
  }
  if (threadIdx.x < 32) vm::tmem_alloc<256>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    uint32_t base = vm::smem_u32(smem);
    uint64_t ad = vm::make_sdesc(base + c.a_off, c.a_lbo, c.a_sbo);
    uint64_t bd = vm::make_sdesc(base + c.b_off, c.b_lbo, c.b_sbo);
    uint32_t id = vm::make_idesc_bf16(c.M, c.N, c.a_mn, c.b_mn);
    vm::mma_bf16_ss(tbase, ad, bd, id, 0);
    vm::mma_commit(&bar);
  }
  vm::mbar_wait(&bar, 0);
  vm::tc_fence_after();
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < 4) {
    for (int n0 = 0; n0 < c.N; n0 += 8) {
      uint32_t r[8];
      vm::tmem_ld8(tbase + ((warp * 32) << 16) + n0, r);
      vm::tmem_ld_wait();
      int m = warp * 32 + lane;
      for (int j = 0; j < 8; ++j) out[m * c.N + n0 + j] = __uint_as_float(r[j]);
    }
  }
  vm::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) vm::tmem_dealloc<256>(tbase);
}

static float bf(bf16 v) { return __bfloat162float(v); }

static int run_case(const char* name, std::vector<bf16>& img, MmaCase c,
                    const std::vector<float>& ref) {
  uint8_t* dimg;
  float* dout;
  int bytes = (int)(img.size() * 2);
  CK(cudaMalloc(&dimg, bytes));
  CK(cudaMalloc(&dout, c.M * c.N * 4));
  CK(cudaMemcpy(dimg, img.data(), bytes, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_single_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  k_single_mma<<<1, 128, bytes>>>(dimg, bytes, c, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> out(c.M * c.N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  for (size_t i = 0; i < out.size(); ++i) {
    maxerr = fmax(maxerr, fabs(out[i] - ref[i]));
    maxref = fmax(maxref, fabs(ref[i]));
  }
  printf("[%s] %s  maxerr=%.3e maxref=%.3e\n", maxerr <= 1e-3 * fmax(1.0, maxref) ? "PASS" : "FAIL",
         name, maxerr, maxref);
  cudaFree(dimg);
  cudaFree(dout);
  return maxerr <= 1e-3 * fmax(1.0, maxref) ? 0 : 1;
}

// A: K-major, stored [2 khalf][R rows][8]; rows shifted by s.  B: K-major [2][N][8].
static int test_kmajor_shift(int s, int N) {
  const int R = 400, M = 128;
  std::vector<bf16> img(2 * R * 8 + 2 * N * 8);
  for (size_t i = 0; i < img.size(); ++i) img[i] = __float2bfloat16((float)((i * 37 % 17) - 8) / 8.f);
  auto A = [&](int r, int k) { return bf(img[(k / 8) * R * 8 + r * 8 + (k % 8)]); };
  int boff = 2 * R * 8;
  auto B = [&](int n, int k) { return bf(img[boff + (k / 8) * N * 8 + n * 8 + (k % 8)]); };
  std::vector<float> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float acc = 0;
      for (int k = 0; k < 16; ++k) acc += A(s + m, k) * B(n, k);
      ref[m * N + n] = acc;
    }
  MmaCase c{(uint32_t)(s * 16), (uint32_t)(R * 16), 128, (uint32_t)(boff * 2), (uint32_t)(N * 16), 128, M, N, 0, 0};
  char name[128];
  snprintf(name, sizeof name, "K-major A row-shift s=%d N=%d", s, N);
  return run_case(name, img, c, ref);
}

// A single plane [R][8] (Cin=8); K half 1 = rows shifted by delta (LBO = 16*delta).
static int test_lbo_tap(int s, int delta) {
  const int R = 400, M = 128, N = 16;
  std::vector<bf16> img(R * 8 + 2 * N * 8);
  for (size_t i = 0; i < img.size(); ++i) img[i] = __float2bfloat16((float)((i * 29 % 13) - 6) / 4.f);
  auto A = [&](int r, int k) { return bf(img[r * 8 + k]); };
  int boff = R * 8;
  auto B = [&](int n, int k) { return bf(img[boff + (k / 8) * N * 8 + n * 8 + (k % 8)]); };
  std::vector<float> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float acc = 0;
      for (int k = 0; k < 8; ++k) acc += A(s + m, k) * B(n, k);
      for (int k = 0; k < 8; ++k) acc += A(s + m + delta, k) * B(n, 8 + k);
      ref[m * N + n] = acc;
    }
  MmaCase c{(uint32_t)(s * 16), (uint32_t)(delta * 16), 128, (uint32_t)(boff * 2), (uint32_t)(N * 16), 128, M, N, 0, 0};
  char name[128];
  snprintf(name, sizeof name, "LBO-as-tap s=%d delta=%d", s, delta);
  return run_case(name, img, c, ref);
}

// MN-major A and B: stored [mn/8][K rows][8].  D[m][n] = sum_k A[k][m] B[k][n].
static int test_mn_major(int M, int N, int shiftk) {
  const int KR = 64;  // K rows available
  std::vector<bf16> img((M / 8) * KR * 8 + (N / 8) * KR * 8);
  for (size_t i = 0; i < img.size(); ++i) img[i] = __float2bfloat16((float)((i * 41 % 19) - 9) / 8.f);
  auto A = [&](int k, int m) { return bf(img[(m / 8) * KR * 8 + k * 8 + (m % 8)]); };
  int boff = (M / 8) * KR * 8;
  auto B = [&](int k, int n) { return bf(img[boff + (n / 8) * KR * 8 + k * 8 + (n % 8)]); };
  std::vector<float> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float acc = 0;
      for (int k = 0; k < 16; ++k) acc += A(k + shiftk, m) * B(k + shiftk, n);
      ref[m * N + n] = acc;
    }
  // MN-major: SBO = distance between 8-element MN groups, LBO = between 8-row K groups
  MmaCase c{(uint32_t)(shiftk * 16), 128, (uint32_t)(KR * 16), (uint32_t)(boff * 2 + shiftk * 16), 128,
            (uint32_t)(KR * 16), M, N, 1, 1};
  char name[128];
  snprintf(name, sizeof name, "MN-major A,B M=%d N=%d kshift=%d", M, N, shiftk);
  return run_case(name, img, c, ref);
}

// ------------------------------------------------------------ throughput
__global__ void k_mma_tput(int N, int iters, int shift_mode, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 160 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    vm::mbar_init(&bar, 1);
    vm::fence_barrier_init();
  }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    uint32_t base = vm::smem_u32(smem);
    const int R = 2048;  // A: [2][R][8] = 64 KB
    uint32_t id = vm::make_idesc_bf16(128, N, 0, 0);
    uint64_t bd = vm::make_sdesc(base + 2 * R * 16, N * 16, 128);
    const int offs[9] = {0, 1, 2, 130, 131, 132, 260, 261, 262};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      int s = shift_mode ? offs[it % 9] : 0;
      uint64_t ad = vm::make_sdesc(base + s * 16, R * 16, 128);
      vm::mma_bf16_ss(tbase + ((it & 1) ? 256 : 0) * (N <= 256 && N * 2 <= 512 ? 1 : 0), ad, bd, id, 1);
    }
    vm::mma_commit(&bar);
    vm::mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  vm::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) vm::tmem_dealloc<512>(tbase);
}

static void tput(int N, int shift_mode, int grid) {
  long long* dcyc;
  CK(cudaMalloc(&dcyc, grid * sizeof(long long)));
  CK(cudaFuncSetAttribute(k_mma_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mma_tput<<<grid, 128, 160 * 1024>>>(N, 100, shift_mode, dcyc);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_mma_tput<<<grid, 128, 160 * 1024>>>(N, iters, shift_mode, dcyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> cyc(grid);
  CK(cudaMemcpy(cyc.data(), dcyc, grid * sizeof(long long), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (auto c : cyc) avg += c;
  avg /= grid;
  double flops = 2.0 * 128 * N * 16 * (double)iters * grid;
  printf("MMA M=128 N=%3d K=16 shift=%d grid=%3d: %.2f cyc/mma  (ideal %.1f)  chip %.1f TFLOP/s\n", N,
         shift_mode, grid, avg / iters, 128.0 * N / 256.0, flops / (ms * 1e-3) / 1e12);
  cudaFree(dcyc);
}

// ------------------------------------------------------------ TMA
__global__ void k_tma(const __grid_constant__ CUtensorMap map2, const __grid_constant__ CUtensorMap map3,
                      int row0, bf16* out2, bf16* out3) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    vm::mbar_init(&bar, 1);
    vm::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    vm::mbar_arrive_expect_tx(&bar, 256 * 16 + 2 * 256 * 16);
    vm::tma_load_2d(smem, &map2, &bar, 0, row0);
    vm::tma_load_3d(smem + 4096, &map3, &bar, 0, row0, 0);
  }
  vm::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) out2[i] = reinterpret_cast<bf16*>(smem)[i];
  for (int i = threadIdx.x; i < 2 * 256 * 8; i += blockDim.x) out3[i] = reinterpret_cast<bf16*>(smem + 4096)[i];
}

static int test_tma() {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  const int ROWS = 1000, CG = 2;
  std::vector<bf16> h(CG * ROWS * 8);
  for (size_t i = 0; i < h.size(); ++i) h[i] = __float2bfloat16((float)(i % 251));
  bf16 *d, *o2, *o3;
  CK(cudaMalloc(&d, h.size() * 2));
  CK(cudaMalloc(&o2, 256 * 8 * 2));
  CK(cudaMalloc(&o3, 2 * 256 * 8 * 2));
  CK(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  CUtensorMap m2, m3;
  cuuint64_t dims2[2] = {8, (cuuint64_t)(CG * ROWS)};
  cuuint64_t str2[1] = {16};
  cuuint32_t box2[2] = {8, 256};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims2, str2, box2, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode2 failed %d\n", r); return 1; }
  cuuint64_t dims3[3] = {8, (cuuint64_t)ROWS, (cuuint64_t)CG};
  cuuint64_t str3[2] = {16, (cuuint64_t)ROWS * 16};
  cuuint32_t box3[3] = {8, 256, 2};
  r = encode(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims3, str3, box3, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode3 failed %d\n", r); return 1; }
  int row0 = 900;  // box runs past ROWS in map3 -> OOB zero fill
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  k_tma<<<1, 128, 64 * 1024>>>(m2, m3, row0, o2, o3);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<bf16> g2(256 * 8), g3(2 * 256 * 8);
  CK(cudaMemcpy(g2.data(), o2, g2.size() * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(g3.data(), o3, g3.size() * 2, cudaMemcpyDeviceToHost));
  int bad2 = 0, bad3 = 0;
  for (int r2 = 0; r2 < 256; ++r2)
    for (int j = 0; j < 8; ++j) {
      int row = row0 + r2;
      float want = row < CG * ROWS ? bf(h[row * 8 + j]) : 0.f;
      if (bf(g2[r2 * 8 + j]) != want) bad2++;
    }
  for (int c = 0; c < 2; ++c)
    for (int r2 = 0; r2 < 256; ++r2)
      for (int j = 0; j < 8; ++j) {
        int row = row0 + r2;
        float want = row < ROWS ? bf(h[(c * ROWS + row) * 8 + j]) : 0.f;
        if (bf(g3[(c * 256 + r2) * 8 + j]) != want) bad3++;
      }
  printf("[%s] TMA 2D box [8,256] bad=%d\n", bad2 ? "FAIL" : "PASS", bad2);
  printf("[%s] TMA 3D box [8,256,2] with OOB fill bad=%d\n", bad3 ? "FAIL" : "PASS", bad3);
  return (bad2 || bad3) ? 1 : 0;
}

int main() {
  int fails = 0;
  for (int s : {0, 1, 2, 3, 7, 8, 9, 130, 262}) fails += test_kmajor_shift(s, 16);
  for (int N : {32, 64, 128, 256}) fails += test_kmajor_shift(5, N);
  for (int d : {1, 2, 3, 130}) fails += test_lbo_tap(3, d);
  fails += test_mn_major(128, 16, 0);
  fails += test_mn_major(128, 32, 8);
  fails += test_mn_major(64, 16, 3);
  fails += test_tma();
  for (int N : {16, 32, 64, 128, 256}) tput(N, 0, 148);
  for (int N : {16, 32, 64}) tput(N, 1, 148);
  tput(16, 0, 1);
  tput(128, 0, 1);
  printf("fails=%d\n", fails);
  return fails ? 1 : 0;
}
