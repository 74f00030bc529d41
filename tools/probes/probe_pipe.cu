// probe_pipe.cu — the conv forward pipeline in isolation: a producer warp bulk-copies
// (A run + weight block) per stage into a ring, the MMA warp waits on `full`, issues 9*MB
// MMAs (M=128, N, K=16, row-shifted A), commits `empty`.  Measures cycles per MMA for
// weight blocks shared by all CTAs (L2 broadcast) vs private per CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_pipe probe_pipe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   vm::smem_u32(dst)), "l"(src), "r"(bytes), "r"(vm::smem_u32(bar))
               : "memory");
}

template <int N, int MB>
__global__ void __launch_bounds__(320, 1) k_pipe(const uint8_t* gA, const uint8_t* gW, int nst, int shared_w,
                                                 int nstages, long long* out, int spin, int Wp, int nacc, int notma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8], fin;
  __shared__ uint32_t tslot;
  const int R = MB * 128 + 2 * Wp + 2;
  const uint32_t a_bytes = (uint32_t)((R + 7) / 8 * 8) * 16;
  const uint32_t b_bytes = 9 * 2 * N * 16;
  const uint32_t stage_bytes = 2 * a_bytes + b_bytes;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) { vm::mbar_init(&full[s], 1); vm::mbar_init(&empty[s], 1); }
    vm::mbar_init(&fin, 1);
    vm::fence_barrier_init();
  }
  if (warp == 1) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  const uint32_t tbase = tslot;
  long long t0 = clock64();
  if (warp == 0) {
    if (vm::elect_one()) {
      int stage = 0; uint32_t ph = 0;
      for (int s = 0; s < nst; ++s) {
        vm::mbar_wait(&empty[stage], ph ^ 1);
        uint8_t* sA = smem + stage * stage_bytes;
        if (notma) {
          vm::mbar_arrive(&full[stage]);
          if (++stage == nstages) { stage = 0; ph ^= 1; }
          continue;
        }
        vm::mbar_arrive_expect_tx(&full[stage], 2 * R * 16 + b_bytes);
        const uint8_t* ga = gA + ((size_t)blockIdx.x * 64 + (s % 64)) * 8192;
        bulk(sA, ga, R * 16, &full[stage]);
        bulk(sA + a_bytes, ga + 4096, R * 16, &full[stage]);
        const uint8_t* gw = gW + (size_t)(s % 24) * b_bytes + (shared_w ? 0 : (size_t)blockIdx.x * 24 * b_bytes);
        bulk(sA + 2 * a_bytes, gw, b_bytes, &full[stage]);
        if (++stage == nstages) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    int stage = 0; uint32_t ph = 0;
    constexpr uint32_t id = vm::make_idesc_bf16(128, N, false, false);
    for (int s = 0; s < nst; ++s) {
      if (!(notma & 4)) vm::mbar_wait(&full[stage], ph);
      if (!(notma & 2)) vm::tc_fence_after();
      if (vm::elect_one()) {
        const uint32_t sA = vm::smem_u32(smem + stage * stage_bytes);
        const uint64_t a0 = vm::make_sdesc(sA, a_bytes, 128);
        const uint64_t b0 = vm::make_sdesc(sA + 2 * a_bytes, N * 16, 128);
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          const uint64_t bd = b0 + (uint64_t)(j * (2 * N * 16 / 16));
          const uint64_t ad = a0 + (uint64_t)((j / 3) * Wp + (j % 3));
#pragma unroll
          for (int i = 0; i < MB; ++i)
            vm::mma_bf16_ss(tbase + (uint32_t)((i * nacc + s % nacc) * N), ad + (uint64_t)(i * 128), bd, id, (s >= nacc || j > 0) ? 1u : 0u);
        }
        vm::mma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == nstages) { stage = 0; ph ^= 1; }
    }
    // wait for the last MMAs
    const int last = (nst - 1) % nstages;
    const uint32_t lph = ((nst - 1) / nstages) & 1;
    vm::mbar_wait(&empty[last], lph);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
    if (threadIdx.x == 32) vm::mbar_arrive(&fin);
  } else if (spin) {
    vm::mbar_wait(&fin, 0);  // idle epilogue warps polling a barrier, as in the conv kernels
  }
  vm::tc_fence_before();
  __syncthreads();
  if (warp == 1) vm::tmem_dealloc<512>(tbase);
}

template <int N, int MB>
void run(int grid, int shared_w, int nstages, int spin = 0, int Wp = 34, int nacc = 1, int notma = 0) {
  static uint8_t *gA = nullptr, *gW = nullptr;
  if (!gA) {
    cudaMalloc(&gA, (size_t)148 * 64 * 8192 + 65536);
    cudaMalloc(&gW, (size_t)148 * 24 * 9 * 2 * 256 * 16);
    cudaMemset(gA, 0x3c, (size_t)148 * 64 * 8192 + 65536);
    cudaMemset(gW, 0x3c, (size_t)148 * 24 * 9 * 2 * 256 * 16);
  }
  long long* d; cudaMalloc(&d, 148 * 8);
  const int R = MB * 128 + 2 * Wp + 2;
  const size_t smem = (size_t)nstages * (2 * ((R + 7) / 8 * 8) * 16 + 9 * 2 * N * 16);
  if (smem > 220 * 1024) { printf("N=%d MB=%d stages=%d: smem too big\n", N, MB, nstages); return; }
  cudaFuncSetAttribute(k_pipe<N, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nst = 240;
  k_pipe<N, MB><<<grid, 320, smem>>>(gA, gW, 24, shared_w, nstages, d, spin, Wp, nacc, notma);
  k_pipe<N, MB><<<grid, 320, smem>>>(gA, gW, nst, shared_w, nstages, d, spin, Wp, nacc, notma);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= grid;
  printf("notma=%d Wp=%d nacc=%d ", notma, Wp, nacc);
  printf("N=%3d MB=%d grid=%3d stages=%d weights %s: %7.1f cyc/mma (%7.0f cyc/stage) %s\n", N, MB, grid, nstages,
         shared_w ? "shared " : "private", avg / (nst * 9.0 * MB), avg / nst, err ? cudaGetErrorString(err) : "");
  cudaFree(d);
}

int main() {
  for (int m : {1, 7}) { run<48, 3>(148, 1, 4, 1, 130, 1, m); run<128, 1>(41, 1, 4, 1, 18, 3, m); run<64, 2>(145, 1, 6, 1, 34, 1, m); }
  return 0;
}
