// probe_tma.cu — L2->SMEM throughput of TMA tensor boxes vs bulk copies (1 CTA/SM, 148 CTAs).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(vm::smem_u32(dst)), "l"(src), "r"(bytes), "r"(vm::smem_u32(bar)) : "memory");
}

// mode 0: bulk copies of `chunk` bytes; mode 1: 2D tensor box {8, rows}; mode 2: box {64, rows/8}
__global__ void k_tma(const __grid_constant__ CUtensorMap m8, const __grid_constant__ CUtensorMap m64,
                      const uint8_t* src, int mode, int chunk, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) vm::mbar_init(&bar[i], 1); vm::fence_barrier_init(); }
  __syncthreads();
  if (mode == 3) {  // all 32 lanes issue bulk copies
    const int lane = threadIdx.x;
    const int per_stage = 32768;
    long long t0 = clock64();
    uint32_t ph[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
      int s = it & 3;
      if (it >= 4) { vm::mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
      __syncwarp();
      if (lane == 0) vm::mbar_arrive_expect_tx(&bar[s], per_stage);
      __syncwarp();
      uint8_t* dst = smem + s * per_stage;
      size_t base = ((size_t)blockIdx.x * 977 + it * 31) % 4096 * 32768;
      for (int off = lane * chunk; off < per_stage; off += 32 * chunk) bulk_load(dst + off, src + base + off, chunk, &bar[s]);
    }
    for (int s = 0; s < 4; ++s) vm::mbar_wait(&bar[s], ph[s]);
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    return;
  }
  if (threadIdx.x != 0) return;
  const int per_stage = 32768;  // bytes per stage
  long long t0 = clock64();
  uint32_t ph[4] = {0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    int s = it & 3;
    if (it >= 4) { vm::mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
    vm::mbar_arrive_expect_tx(&bar[s], per_stage);
    uint8_t* dst = smem + s * per_stage;
    size_t base = ((size_t)blockIdx.x * 977 + it * 31) % 4096 * 32768;
    if (mode == 0) {
      for (int off = 0; off < per_stage; off += chunk) bulk_load(dst + off, src + base + off, chunk, &bar[s]);
    } else if (mode == 1) {
      int rows = chunk / 16;
      for (int off = 0; off < per_stage; off += chunk)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(vm::smem_u32(dst + off)), "l"(&m8), "r"(0), "r"((int)((base + off) / 16)), "r"(vm::smem_u32(&bar[s])) : "memory");
      (void)rows;
    } else {
      for (int off = 0; off < per_stage; off += chunk)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(vm::smem_u32(dst + off)), "l"(&m64), "r"(0), "r"((int)((base + off) / 128)), "r"(vm::smem_u32(&bar[s])) : "memory");
    }
  }
  for (int s = 0; s < 4; ++s) { vm::mbar_wait(&bar[s], ph[s]); }
  cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  size_t bytes = (size_t)4096 * 32768 + (1 << 20);
  uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  long long* cyc; cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  int chunks[] = {512, 1024, 2048, 4096, 8192};
  for (int mode = 0; mode < 4; ++mode)
    for (int chunk : chunks) {
      CUtensorMap m8, m64;
      cuuint64_t d8[2] = {8, bytes / 16}; cuuint64_t s8[1] = {16}; cuuint32_t b8[2] = {8, (cuuint32_t)(chunk / 16 > 256 ? 256 : chunk / 16)};
      cuuint64_t d64[2] = {64, bytes / 128}; cuuint64_t s64[1] = {128}; cuuint32_t b64[2] = {64, (cuuint32_t)(chunk / 128)};
      cuuint32_t es[2] = {1, 1};
      enc(&m8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, d8, s8, b8, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      enc(&m64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, d64, s64, b64, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (mode == 1 && chunk > 4096) continue;
      int iters = 400;
      k_tma<<<148, 32, 140 * 1024>>>(m8, m64, src, mode, chunk, 8, cyc);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_tma<<<148, 32, 140 * 1024>>>(m8, m64, src, mode, chunk, iters, cyc);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (auto c : h) avg += c; avg /= 148;
      double tot = 148.0 * iters * 32768;
      printf("mode=%d (%s) chunk=%5d: %.1f B/cyc/SM, chip %.2f TB/s %s\n", mode,
             mode == 0 ? "bulk" : mode == 1 ? "box8x16B" : mode == 2 ? "box128B" : "bulk32lanes", chunk, iters * 32768.0 / avg,
             tot / (ms * 1e-3) / 1e12, err ? cudaGetErrorString(err) : "");
    }
  return 0;
}
