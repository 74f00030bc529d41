// probe_sweep_mma.cu — the kd-stacked sweep kernel's MMA stream alone (no TMA, no epilogue):
// per input plane, 9 taps x MB tiles of N = 3*Nc into a TMEM ring (blocks advance by one per
// plane, split at the ring end), first tap split into N=2Nc (acc) + N=Nc (overwrite).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_sweep_mma probe_sweep_mma.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

template <int MB>
__global__ void k(int planes, int ring, int Nc, int split_first, int Wp, long long* out, int fixb, int fixd, int fixa, int tsov) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 160 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<int4*>(smem + i) = make_int4(0x3c003c00, 0x3c003c00, 0, 0);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) { vm::mbar_init(&bar, 1); vm::fence_barrier_init(); }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x < 32) {
    const uint32_t base = vm::smem_u32(smem);
    const uint32_t a_bytes = ((MB * 128 + 2 * Wp + 2) * 16 + 127) & ~127u;
    const uint32_t wblk = 2 * 3 * Nc * 16;
    const uint32_t id1 = vm::make_idesc_bf16(128, Nc, false, false), id2 = vm::make_idesc_bf16(128, 2 * Nc, false, false),
                   id3 = vm::make_idesc_bf16(128, 3 * Nc, false, false);
    const uint32_t tstride = tsov ? tsov : ring * Nc;
    long long t0 = clock64();
    if (vm::elect_one()) {
      for (int n = 0; n < planes; ++n) {
        const uint32_t pos = fixd ? 0 : n % ring;
        const uint32_t sA = base + 64 * 1024 + (n & 1) * 2 * a_bytes;
        const uint64_t a0 = vm::make_sdesc(sA, a_bytes, 128);
        const uint64_t b0 = vm::make_sdesc(base, 3 * Nc * 16, 128);
        for (int j = 0; j < 9; ++j) {
          const uint64_t bd = b0 + (uint64_t)(fixb ? 0 : j * (wblk >> 4));
          const uint64_t ad = a0 + (uint64_t)(fixa ? 0 : (j / 3) * Wp + (j % 3));
#pragma unroll
          for (int t = 0; t < MB; ++t) {
            const uint32_t dt = tbase + t * tstride;
            const uint64_t at = ad + (uint64_t)(t * 128);
            if (j == 0 && split_first) {
              if (pos + 2 < (uint32_t)ring) {
                vm::mma_bf16_ss(dt + pos * Nc, at, bd, id2, 1u);
                vm::mma_bf16_ss(dt + (pos + 2) * Nc, at, bd + 2 * Nc, id1, 0u);
              } else {
                vm::mma_bf16_ss(dt + 0, at, bd, id1, 1u);
              }
            } else if (pos + 3 <= (uint32_t)ring) {
              vm::mma_bf16_ss(dt + pos * Nc, at, bd, id3, 1u);
            } else {
              vm::mma_bf16_ss(dt, at, bd, id1, 1u);
              vm::mma_bf16_ss(dt + Nc, at, bd + Nc, id2, 1u);
            }
          }
        }
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

template <int MB>
void run(int ring, int Nc, int split_first, int fixb = 0, int fixd = 0, int fixa = 0, int tsov = 0) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int planes = 200;
  cudaFuncSetAttribute(k<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  k<MB><<<148, 128, 160 * 1024>>>(4, ring, Nc, split_first, 130, d, fixb, fixd, fixa, tsov);
  k<MB><<<148, 128, 160 * 1024>>>(planes, ring, Nc, split_first, 130, d, fixb, fixd, fixa, tsov);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= 148;
  const double nm = planes * 9.0 * MB;
  printf("tstride=%3d fixB=%d fixD=%d fixA=%d ", tsov, fixb, fixd, fixa);
  printf("MB=%d ring=%2d Nc=%d split_first=%d: %7.1f cyc/plane  %5.1f cyc per tile-tap  %s\n", MB, ring, Nc, split_first,
         avg / planes, avg / nm, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  run<3>(10, 16, 0, 1, 1, 1, 48); run<3>(10, 16, 0, 1, 1, 1, 64); run<3>(10, 16, 0, 1, 1, 1, 128); run<3>(10, 16, 0, 1, 1, 1, 160);
  run<3>(10, 16, 0, 0, 0, 0, 0);
  return 0;
}
