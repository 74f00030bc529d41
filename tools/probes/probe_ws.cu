// probe_ws.cu — does tcgen05.mma.ws with the B collector buffer (fill / use / lastuse) make the
// kd weight gradient's three kw MMAs per K step cheaper?  They share B (gy) and differ in A
// (a +16 B row shift).  Prints cycles per MMA for plain SS MMAs and .ws MMAs, M = 64,
// MN-major A and B (the kd kernel's operand layout), 3 independent accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_ws probe_ws.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../../paper_1909_03108_b200/csrc/sm100.cuh"

__device__ __forceinline__ void mma_ws(int mode, uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  // mode 0 fill, 1 use, 2 lastuse, 3 discard
  if (mode == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::fill [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else if (mode == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::use [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else if (mode == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::lastuse [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::discard [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

// variant 0: plain SS x3 (same B); 1: ws fill/use/lastuse; 2: ws discard x3 (no reuse)
template <int N, int VAR, int M>
__global__ void k_tput(int iters, long long* cycles) {
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
    constexpr uint32_t id = vm::make_idesc_bf16(M, N, true, true);
    const uint64_t bd0 = vm::make_sdesc(base + 96 * 1024, 128, 256 * 16);
    const uint64_t ad0 = vm::make_sdesc(base, 128, 130 * 16);
    long long t0 = clock64();
    if (vm::elect_one()) {
      for (int it = 0; it < iters; it += 3) {
        const int kk = (it / 3) & 7;
        const uint64_t bd = bd0 + (uint64_t)(kk * 16);
        const uint64_t ad = ad0 + (uint64_t)(kk * 16);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const uint32_t d = tbase + (uint32_t)(s * N);
          if (VAR == 0) vm::mma_bf16_ss(d, ad + s, bd, id, 1);
          else if (VAR == 1) mma_ws(s == 0 ? 0 : s == 2 ? 2 : 1, d, ad + s, bd, id, 1);
          else mma_ws(3, d, ad + s, bd, id, 1);
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

template <int N, int VAR, int M = 64>
void run() {
  const int grid = 148, iters = 3 * 8 * 400;
  long long* d; cudaMalloc(&d, grid * 8);
  cudaFuncSetAttribute(k_tput<N, VAR, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_tput<N, VAR, M><<<grid, 128, 200 * 1024>>>(24, d);
  k_tput<N, VAR, M><<<grid, 128, 200 * 1024>>>(iters, d);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<long long> h(grid); cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto x : h) avg += x; avg /= grid;
  const char* nm[3] = {"plain SS        ", "ws fill/use/last", "ws discard      "};
  printf("M=%3d N=%3d %s: %6.2f cyc/mma  %s\n", M, N, nm[VAR], avg / iters, err ? cudaGetErrorString(err) : "ok");
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int c = argc > 1 ? atoi(argv[1]) : 0;
  switch (c) {
    case 0: run<48, 0>(); break;
    case 1: run<64, 0>(); break;
    case 2: run<48, 1>(); break;
    case 3: run<64, 1>(); break;
    case 4: run<64, 2>(); break;
    case 5: run<128, 1>(); break;
    case 6: run<64, 1, 128>(); break;
    case 7: run<128, 1, 128>(); break;
    case 8: run<256, 1, 128>(); break;
    case 9: run<128, 0, 128>(); break;
    case 10: run<64, 1, 32>(); break;
    case 11: run<96, 0>(); break;
  }
  return 0;
}
