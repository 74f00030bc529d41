// probe_operand_change.cu — cost of an SS-mode tcgen05.mma (M=128, K=16) as a function of how
// often its A and B operands change: every MMA, every R-th MMA, or never.  3 accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_operand_change probe_operand_change.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int N>
__global__ void k(int iters, int a_every, int b_every, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 200 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0x3c003c00, 0x3c003c00, 0x3c003c00, 0x3c003c00);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) { vm::mbar_init(&bar, 1); vm::fence_barrier_init(); }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x < 32) {
    const uint32_t base = vm::smem_u32(smem);
    constexpr uint32_t id = vm::make_idesc_bf16(128, N, false, false);
    const uint64_t a0 = vm::make_sdesc(base, 48 * 1024, 128);          // A region [0, 96 KB)
    const uint64_t b0 = vm::make_sdesc(base + 112 * 1024, N * 16, 128);  // B region [112 KB, ..)
    long long t0 = clock64();
    if (vm::elect_one()) {
      uint32_t ai = 0, bi = 0;
      for (int it = 0; it < iters; ++it) {
        // A steps by 64 rows (1 KB) within 40 KB, B by N*32 B within 80 KB
        const uint64_t ad = a0 + (uint64_t)((ai % 40) * 64);
        const uint64_t bd = b0 + (uint64_t)((bi % (80 * 1024 / (N * 32))) * (N * 2));
        vm::mma_bf16_ss(tbase + (uint32_t)((it % 3) * N), ad, bd, id, 1u);
        if (a_every && (it + 1) % a_every == 0) ++ai;
        if (b_every && (it + 1) % b_every == 0) ++bi;
      }
      vm::mma_commit(&bar);
    }
    __syncwarp();
    vm::mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  vm::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) vm::tmem_dealloc<512>(tbase);
}

template <int N>
void run(int a_every, int b_every) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int iters = 6000;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<N><<<148, 128, 200 * 1024>>>(30, a_every, b_every, d);
  k<N><<<148, 128, 200 * 1024>>>(iters, a_every, b_every, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= 148;
  printf("N=%3d A changes every %d, B changes every %d MMAs (0 = never): %6.1f cyc/mma %s\n", N, a_every, b_every,
         avg / iters, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  run<48>(0, 0); run<48>(1, 0); run<48>(0, 1); run<48>(1, 1); run<48>(1, 3); run<48>(3, 1); run<48>(1, 9);
  run<128>(0, 0); run<128>(1, 0); run<128>(0, 1); run<128>(1, 1); run<128>(1, 3);
  run<16>(1, 0); run<16>(1, 1); run<16>(0, 1);
  return 0;
}
