// probe_tput2.cu — tcgen05.mma issue-rate vs accumulator-chain count (SS, M=128, K=16).
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int N, int CHAINS>
__global__ void k_tput(int iters, int shift, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 96 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) { vm::mbar_init(&bar, 1); vm::fence_barrier_init(); }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  uint32_t tbase = tslot;
  if (threadIdx.x < 32) {   // whole warp enters; one elected lane issues
    uint32_t base = vm::smem_u32(smem);
    const int R = 1500;
    constexpr uint32_t id = vm::make_idesc_bf16(128, N, false, false);
    uint64_t bd = vm::make_sdesc(base + 2 * R * 16, N * 16, 128);
    uint64_t ad0 = vm::make_sdesc(base, R * 16, 128);
    long long t0 = clock64();
    if (vm::elect_one()) {
      for (int it = 0; it < iters; it += CHAINS) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
          uint64_t ad = ad0 + (shift ? (uint64_t)(c * 126 + (it % 3) * 130) : 0ull);  // row shifts like the conv
          vm::mma_bf16_ss(tbase + (uint32_t)(c * N), ad, bd, id, 1);
        }
      }
      vm::mma_commit(&bar);
    }
    __syncwarp();
    vm::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  vm::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) vm::tmem_dealloc<512>(tbase);
}

template <int N, int CHAINS>
void run(int shift) {
  const int grid = 148, iters = 24000;
  long long* d; cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(k_tput<N, CHAINS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  k_tput<N, CHAINS><<<grid, 128, 96 * 1024>>>(96, shift, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_tput<N, CHAINS><<<grid, 128, 96 * 1024>>>(iters, shift, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= grid;
  printf("N=%3d chains=%2d shift=%d: %6.2f cyc/mma (ideal %5.1f) chip %7.1f TFLOP/s %s\n", N, CHAINS, shift,
         avg / iters, 128.0 * N / 256, 2.0 * 128 * N * 16 * iters * grid / (ms * 1e-3) / 1e12,
         err ? cudaGetErrorString(err) : "");
  cudaFree(d);
}

int main() {
  run<16, 5>(0); run<16, 5>(1);
  run<48, 5>(0); run<48, 5>(1);
  run<96, 2>(0); run<96, 2>(1);
  run<32, 5>(0); run<32, 5>(1);
  run<64, 4>(0); run<64, 4>(1);
  return 0;
}
