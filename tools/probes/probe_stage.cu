// probe_stage.cu — per-stage cost of the MMA warp's pipeline protocol (wait full -> fence ->
// elect -> K MMAs -> commit empty), with a producer warp that only arrives (no TMA).
// cycles/stage = overhead + K * mma: fit from K = 1, 3, 9, 27.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_stage probe_stage.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int K>
__global__ void __launch_bounds__(128, 1) k(int nst, int nstages, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x * 16; i < 64 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0x3c003c00, 0, 0x3c003c00, 0);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) { vm::mbar_init(&full[s], 1); vm::mbar_init(&empty[s], 1); }
    vm::fence_barrier_init();
  }
  if (warp == 1) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    if (vm::elect_one()) {
      int stage = 0; uint32_t ph = 0;
      for (int s = 0; s < nst; ++s) {
        vm::mbar_wait(&empty[stage], ph ^ 1);
        vm::mbar_arrive(&full[stage]);
        if (++stage == nstages) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t base = vm::smem_u32(smem);
    constexpr uint32_t id = vm::make_idesc_bf16(128, 48, false, false);
    int stage = 0; uint32_t ph = 0;
    long long t0 = clock64();
    for (int s = 0; s < nst; ++s) {
      vm::mbar_wait(&full[stage], ph);
      vm::tc_fence_after();
      if (vm::elect_one()) {
        const uint64_t a0 = vm::make_sdesc(base + stage * 4096, 16384, 128);
        const uint64_t b0 = vm::make_sdesc(base + 40960, 48 * 16, 128);
#pragma unroll
        for (int j = 0; j < K; ++j)
          vm::mma_bf16_ss(tbase + (uint32_t)((j % 3) * 48), a0 + (uint64_t)(j % 9), b0, id, 1u);
        vm::mma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == nstages) { stage = 0; ph ^= 1; }
    }
    const int last = (nst - 1) % nstages;
    vm::mbar_wait(&empty[last], ((nst - 1) / nstages) & 1);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
  vm::tc_fence_before();
  __syncthreads();
  if (warp == 1) vm::tmem_dealloc<512>(tbase);
}

template <int K>
void run(int nstages) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int nst = 2000;
  cudaFuncSetAttribute(k<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<K><<<148, 128, 64 * 1024>>>(50, nstages, d);
  k<K><<<148, 128, 64 * 1024>>>(nst, nstages, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= 148;
  printf("K=%2d MMAs/stage (N=48), %d stages: %7.1f cycles/stage = %6.1f per MMA %s\n", K, nstages, avg / nst,
         avg / nst / K, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  for (int ns : {2, 4, 8}) { run<1>(ns); run<3>(ns); run<9>(ns); run<27>(ns); }
  return 0;
}
