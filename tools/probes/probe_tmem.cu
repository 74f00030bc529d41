// probe_tmem.cu — tcgen05.ld (TMEM -> registers) throughput with 4 / 8 warps per CTA.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

__global__ void k_ld(int iters, int nwarps_active, long long* cyc, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) vm::tmem_alloc<512>(&tslot);
  vm::tc_fence_before();
  __syncthreads();
  vm::tc_fence_after();
  uint32_t t = tslot;
  float acc = 0.f;
  long long t0 = clock64();
  if (warp < nwarps_active) {
    const int q = warp & 3;
    for (int it = 0; it < iters; it += 4) {
      uint32_t r[4][16];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        vm::tmem_ld16(t + ((uint32_t)(q * 32) << 16) + (uint32_t)(((it + j) * 16) & 511), r[j]);
      vm::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc += __uint_as_float(r[j][e]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  vm::tc_fence_before();
  __syncthreads();
  if (warp == 0) vm::tmem_dealloc<512>(t);
}

int main() {
  long long* cyc; float* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 512 * 4);
  for (int nw : {4, 8, 16}) {
    const int iters = 4096;
    k_ld<<<148, nw * 32>>>(iters, nw, cyc, sink);
    cudaDeviceSynchronize();
    k_ld<<<148, nw * 32>>>(iters, nw, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (auto c : h) avg += c; avg /= 148;
    double bytes = (double)nw * 32 * 16 * 4 * iters;
    printf("warps=%2d: %.1f B/cyc/SM TMEM->RF (%.1f cyc per warp-ld x16) %s\n", nw, bytes / avg, avg / iters,
           e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
