// probe_m64.cu — where does tcgen05.mma (M=64, cta_group::1) put accumulator row m in TMEM?
// A[m][0] = m + 1 (K-major), B[0][0] = 1 and B[8][0] = 1000: D[m][0] = m + 1, D[m][8] = 1000(m+1).
// Prints, for every TMEM lane, the non-zero columns among 0..15 after the MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_m64 probe_m64.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

__global__ void k_probe(float* out) {
  __shared__ __align__(1024) uint8_t smem[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* Bm = reinterpret_cast<__nv_bfloat16*>(smem + 8192);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) A[i] = __float2bfloat16(0.f);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) Bm[i] = __float2bfloat16(0.f);
  __syncthreads();
  // K-major, SWIZZLE_NONE: row m's first 8 K elements at m*16 B (8-row core matrices, SBO = 128)
  if (threadIdx.x < 64) A[threadIdx.x * 8] = __float2bfloat16((float)(threadIdx.x + 1));
  if (threadIdx.x == 0) Bm[0] = __float2bfloat16(1.f);
  if (threadIdx.x == 1) Bm[8 * 8] = __float2bfloat16(1000.f);
  vm::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    vm::mbar_init(&bar, 1);
    vm::fence_barrier_init();
  }
  if (threadIdx.x < 32) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x < 32) {
    if (vm::elect_one()) {
      const uint64_t ad = vm::make_sdesc(vm::smem_u32(A), 64 * 16, 128);
      const uint64_t bd = vm::make_sdesc(vm::smem_u32(Bm), 16 * 16, 128);
      vm::mma_bf16_ss(tbase, ad, bd, vm::make_idesc_bf16(64, 16, false, false), 0);
      vm::mma_commit(&bar);
    }
    __syncwarp();
  }
  vm::mbar_wait(&bar, 0);
  vm::tc_fence_after();
  const int w = threadIdx.x / 32;
  uint32_t r[16];
  vm::tmem_ld16(tbase + ((uint32_t)(w * 32) << 16), r);
  vm::tmem_ld_wait();
  for (int c = 0; c < 16; ++c) out[threadIdx.x * 16 + c] = __uint_as_float(r[c]);
  vm::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) vm::tmem_dealloc<512>(tbase);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 16 * 4);
  k_probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  static float h[128 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  for (int l = 0; l < 128; ++l) {
    printf("lane %3d:", l);
    for (int c = 0; c < 16; ++c)
      if (h[l * 16 + c] != 0.f) printf(" c%d=%g", c, h[l * 16 + c]);
    printf("\n");
  }
  return 0;
}
