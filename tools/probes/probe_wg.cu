// probe_wg.cu — the kd-along-N wgrad MMA loop in isolation: per K step (16 anchors) three
// MMAs (kw = A start +0/+1/+2 rows) into three accumulators, A/B MN-major, B advancing 16 rows
// per K step.  Variants: B fixed vs advancing, M = 64 / 128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_wg probe_wg.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int M, int N>
__global__ void k_wg(int stages, int badv, int aadv, long long* cycles) {
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
    const uint32_t base = vm::smem_u32(smem);
    const uint32_t GS = 130 * 16, KS = 128;
    constexpr uint32_t id = vm::make_idesc_bf16(M, N, true, true);
    long long t0 = clock64();
    if (vm::elect_one()) {
      for (int s = 0; s < stages; ++s) {
        const uint32_t sb = base + (uint32_t)(s & 1) * 96 * 1024;
        const uint64_t b0 = vm::make_sdesc(sb + 64 * 1024, 128, KS * 16);
        const uint64_t a0 = vm::make_sdesc(sb, 128, GS);
#pragma unroll 1
        for (int kk = 0; kk < (int)KS / 16; ++kk) {
          const uint64_t bd = b0 + (uint64_t)(badv ? kk * 16 : 0);
          const uint64_t ad = a0 + (uint64_t)(aadv ? kk * 16 : 0);
          vm::mma_bf16_ss(tbase, ad, bd, id, 1);
          vm::mma_bf16_ss(tbase + N, ad + 1, bd, id, 1);
          vm::mma_bf16_ss(tbase + 2 * N, ad + 2, bd, id, 1);
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

template <int M, int N>
void run(int badv, int aadv) {
  const int grid = 148, stages = 400;
  long long* d; cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(k_wg<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_wg<M, N><<<grid, 128, 200 * 1024>>>(4, badv, aadv, d);
  k_wg<M, N><<<grid, 128, 200 * 1024>>>(stages, badv, aadv, d);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= grid;
  printf("M=%3d N=%3d B %s A %s: %6.2f cyc/mma %s\n", M, N, badv ? "advancing" : "fixed    ",
         aadv ? "advancing" : "fixed    ", avg / (stages * 24.0), err ? cudaGetErrorString(err) : "");
  cudaFree(d);
}

int main() {
  for (int badv : {0, 1})
    for (int aadv : {0, 1}) { run<128, 48>(badv, aadv); run<64, 48>(badv, aadv); run<128, 16>(badv, aadv); }
  return 0;
}
