// probe_tput5.cu — SS-mode tcgen05.mma cost vs A start-address alignment (row-shifted
// K-major A, 16 B rows) and N, with the A start cycling over 9 "taps" like the conv kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_tput5 probe_tput5.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int N, bool MN, int M = 128>
__global__ void k_tput(int iters, int wp, int chains, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 200 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0, 0, 0, 0);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) { vm::mbar_init(&bar, 1); vm::fence_barrier_init(); }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  uint32_t tbase = tslot;
  if (threadIdx.x < 32) {
    uint32_t base = vm::smem_u32(smem);
    const int R = 4096;  // rows per K half (64 KB)
    constexpr uint32_t id = vm::make_idesc_bf16(M, N, MN, MN);
    // K-major: LBO = K-half distance, SBO = 128; MN-major: LBO = 128 (8-row K groups), SBO = MN-group stride
    uint64_t bd = MN ? vm::make_sdesc(base + 64 * 1024, 128, 256 * 16) : vm::make_sdesc(base + 2 * R * 16, N * 16, 128);
    uint64_t ad0 = MN ? vm::make_sdesc(base, 128, (uint32_t)wp * 16 > 0 ? (uint32_t)wp * 16 : 2048) : vm::make_sdesc(base, R * 16, 128);
    long long t0 = clock64();
    if (vm::elect_one()) {
      for (int it = 0; it < iters; it += 9 * chains) {
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          const uint64_t ad = ad0 + (uint64_t)((j / 3) * wp + (j % 3) * (wp > 0 ? 1 : 0));
          for (int c = 0; c < chains; ++c)
            vm::mma_bf16_ss(tbase + (uint32_t)(c * N), ad + (uint64_t)(c * 128), bd, id, 1);
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

template <int N, bool MN = false, int M = 128>
void run(int wp, int chains) {
  const int grid = 148, iters = 9 * 24 * 100;
  long long* d; cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(k_tput<N, MN, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_tput<N, MN, M><<<grid, 128, 200 * 1024>>>(9 * chains, wp, chains, d);
  k_tput<N, MN, M><<<grid, 128, 200 * 1024>>>(iters, wp, chains, d);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= grid;
  printf("M=%d %s N=%3d wp=%3d chains=%d: %6.2f cyc/mma  %s\n", M, MN ? "MN-major" : "K-major ", N, wp, chains,
         avg / iters, err ? cudaGetErrorString(err) : "");
  cudaFree(d);
}

int main() {
  for (int chains : {1, 3, 4}) {
    run<48, true, 64>(130, chains); run<96, true, 64>(130, chains); run<48, true, 128>(130, chains);
    run<16, false, 64>(130, chains); run<48, false, 64>(130, chains); run<96, false, 64>(130, chains);
  }
  return 0;
}
