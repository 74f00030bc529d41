// probe_wg.cu — the kd-along-N wgrad MMA loop in isolation: per K step (16 anchors) three
// MMAs (kw = A start +0/+1/+2 rows) into three accumulators, A/B MN-major, B advancing 16 rows
// per K step.  Variants: B fixed vs advancing, M = 64 / 128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_wg probe_wg.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int M, int N>
__global__ void k_wg(int stages, int badv, int aadv, int rnd, long long* cycles, const uint8_t* gsrc, int tma_kb,
                     int fence) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 4; i < 200 * 1024; i += blockDim.x * 4) {
    uint32_t h = (uint32_t)i * 2654435761u + 12345u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    // two bf16 in [-1, 1): sign/exponent 0x3F (1.x) or 0xBF, random mantissa
    const uint32_t lo = ((h & 1u) ? 0xBF00u : 0x3F00u) | ((h >> 1) & 0x7Fu);
    const uint32_t hi = ((h & 256u) ? 0xBF00u : 0x3F00u) | ((h >> 9) & 0x7Fu);
    *reinterpret_cast<uint32_t*>(smem + i) = rnd ? (hi << 16 | lo) : 0u;
  }
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) { vm::mbar_init(&bar, 1); vm::fence_barrier_init(); }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  uint32_t tbase = tslot;
  __shared__ uint64_t tbar, cbar[2];
  __shared__ volatile int done;
  if (threadIdx.x == 0) { vm::mbar_init(&tbar, 1); vm::mbar_init(&cbar[0], 1); vm::mbar_init(&cbar[1], 1); done = 0; vm::fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x >= 32 && threadIdx.x < 64 && tma_kb > 0) {
    // concurrent TMA traffic: bulk copies of tma_kb KB into smem[192 KB ..) in a loop
    uint32_t ph = 0;
    while (!done) {
      if (threadIdx.x == 32) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(vm::smem_u32(&tbar)), "r"(tma_kb * 1024) : "memory");
        for (int c = 0; c < tma_kb; c += 8)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(vm::smem_u32(smem + 150 * 1024)),
                       "l"(gsrc + (size_t)blockIdx.x * 65536 + c * 1024), "r"(8192), "r"(vm::smem_u32(&tbar)) : "memory");
      }
      __syncwarp();
      vm::mbar_wait(&tbar, ph);
      ph ^= 1;
    }
  }
  if (threadIdx.x < 32) {
    const uint32_t base = vm::smem_u32(smem);
    const uint32_t GS = 130 * 16, KS = 128;
    constexpr uint32_t id = vm::make_idesc_bf16(M, N, true, true);
    long long t0 = clock64();
    if (vm::elect_one()) {
      for (int s = 0; s < stages; ++s) {
        if (fence & 1) vm::tc_fence_after();
        if (fence & 2) vm::mma_commit(&cbar[s & 1]);
        const uint32_t sb = base + (uint32_t)(s & 1) * 64 * 1024;
        const uint64_t b0 = vm::make_sdesc(sb + 40 * 1024, 128, KS * 16);
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
    if (threadIdx.x == 0) done = 1;
  }
  vm::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) vm::tmem_dealloc<512>(tbase);
}

template <int M, int N>
void run(int badv, int aadv, int rnd = 0, int tma_kb = 0, int fence = 0) {
  static uint8_t* gsrc = nullptr;
  if (!gsrc) { cudaMalloc(&gsrc, 148 * 65536 + 65536); cudaMemset(gsrc, 0, 148 * 65536 + 65536); }
  const int grid = 148, stages = 400;
  long long* d; cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(k_wg<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_wg<M, N><<<grid, 128, 200 * 1024>>>(4, badv, aadv, rnd, d, gsrc, tma_kb, fence);
  k_wg<M, N><<<grid, 128, 200 * 1024>>>(stages, badv, aadv, rnd, d, gsrc, tma_kb, fence);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= grid;
  printf("fence %d tma %2d KB/round ", fence, tma_kb);
  printf("%s M=%3d N=%3d B %s A %s: %6.2f cyc/mma %s\n", rnd ? "random" : "zeros ", M, N, badv ? "advancing" : "fixed    ",
         aadv ? "advancing" : "fixed    ", avg / (stages * 24.0), err ? cudaGetErrorString(err) : "");
  cudaFree(d);
}

int main() {
  for (int f : {0, 1, 2, 3}) { run<128, 48>(1, 1, 1, 0, f); run<64, 48>(1, 1, 1, 0, f); run<128, 128>(1, 1, 1, 0, f); }
  return 0;
}
