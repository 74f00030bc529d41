// vm_common.cuh — shared helpers of libvoxmesh_sm100: error plumbing, dtype
// traits, slab geometry.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/vm_api.h"

namespace vm {

void set_error(const char* fmt, ...);
int grid_for(int64_t work, int threads);  // grid-stride grid, capped at 8 x #SMs

#define VM_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::vm::set_error(__VA_ARGS__);  \
      return (code);                 \
    }                                \
  } while (0)

void count_launches(int n);  // bookkeeping for vm_launch_count()

inline int launch_status(const char* what, int nlaunch = 1) {
  count_launches(nlaunch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return static_cast<int>(e);
  }
  return VM_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (PDL).  A kernel launched by launch_pdl may start while the
// previous kernel on its stream is still running: it must call pdl_wait() before its first
// global-memory access (read or write), and calls pdl_trigger() to let the NEXT kernel's
// CTAs be scheduled (prologue: barrier init, TMEM alloc) before this one finishes.  Both are
// no-ops when the kernel was launched without the attribute.  vm_set_pdl(0) turns it off.
bool pdl_enabled();
bool pdl_late();  // mode 2: kernels skip the early trigger (dependents launch as CTAs exit)
constexpr unsigned kFlagPdlLate = 1u << 8;  // conv params flag bit set from pdl_late()
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  if (!pdl_enabled()) {
    kern<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline int dtype_bytes(int dt) {
  switch (dt) {
    case VM_F32: return 4;
    case VM_BF16: return 2;
    case VM_F64: return 8;
    case VM_U8: return 1;
  }
  return 0;
}

template <typename T> struct Cvt;
template <> struct Cvt<float> {
  __device__ __forceinline__ static float to_f(float v) { return v; }
  __device__ __forceinline__ static float from_f(float v) { return v; }
};
template <> struct Cvt<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

// Geometry of a channel-blocked padded slab [B][CG][Dp][Hp][Wp][8].
struct Slab {
  int64_t bstride;  // elements between samples
  int CG, D, H, W, m;
  // floor(2^32 / d) + 1 for W, H, D: voxel-index decomposition by multiply-high instead of
  // runtime division (the HBM-bound kernels are issue-bound otherwise); set by make_slab()
  uint32_t mW = 0, mH = 0, mD = 0;
  __host__ __device__ int Dp() const { return D + 2 * m; }
  __host__ __device__ int Hp() const { return H + 2 * m; }
  __host__ __device__ int Wp() const { return W + 2 * m; }
  __host__ __device__ int64_t plane() const { return (int64_t)Dp() * Hp() * Wp() * 8; }
  // element offset of channel-block (b, cg) at interior voxel (d, h, w)
  __host__ __device__ int64_t at(int b, int cg, int d, int h, int w) const {
    return b * bstride + cg * plane() + ((((int64_t)(d + m) * Hp()) + (h + m)) * Wp() + (w + m)) * 8;
  }
};

inline uint32_t fastdiv_magic(uint32_t d) { return (uint32_t)(0x100000000ULL / d) + 1u; }
// q = n / d for n < 2^31, d < 2^16: multiply-high estimate plus one correction step
__device__ __forceinline__ uint32_t fastdiv(uint32_t n, uint32_t d, uint32_t magic) {
  uint32_t q = __umulhi(n, magic);
  if (q * d > n) --q;
  return q;
}
inline Slab make_slab(int64_t bstride, int CG, int D, int H, int W, int m) {
  Slab s{bstride, CG, D, H, W, m};
  s.mW = fastdiv_magic((uint32_t)W);
  s.mH = fastdiv_magic((uint32_t)H);
  s.mD = fastdiv_magic((uint32_t)D);
  return s;
}

size_t bias_grad_ws_bytes(int64_t nvox, int Cout);
int bias_grad_bf16(const void* gy, int64_t gy_bstride, float* gb, float* ws, int B, int Cout, int D,
                   int H, int W, cudaStream_t st);
int bias_grad_partial_bf16(const void* gy, int64_t gy_bstride, float* ws, int B, int Cout, int D, int H, int W,
                           cudaStream_t st, int* nsplit);

inline int64_t default_bstride(int C, int D, int H, int W, int m) {
  return (int64_t)((C + 7) / 8) * (D + 2 * m) * (H + 2 * m) * (W + 2 * m) * 8;
}


// ------------------------------------------------------------------ fused peer-memory halo
// (vm_halo_link, include/vm_api.h): producer-side boundary-layer stores into the neighbours'
// slabs + one system-scope publish per kernel; consumer-side wait for the own margins.
struct HaloLink {
  __nv_bfloat16* lo;  // lo neighbour's copy of the output slab (its layer D+1 receives our layer 1)
  __nv_bfloat16* hi;  // hi neighbour's copy (its layer 0 receives our layer D)
  int* lo_flag;
  int* hi_flag;
  unsigned* counter;
  const int* wait_own;
  int wait_lo, wait_hi;
  const int* epoch;
};

inline HaloLink halo_link_of(const vm_halo_link* l) {
  HaloLink h{};
  if (l) {
    h.lo = static_cast<__nv_bfloat16*>(l->push_lo), h.hi = static_cast<__nv_bfloat16*>(l->push_hi);
    h.lo_flag = l->lo_flag, h.hi_flag = l->hi_flag, h.counter = l->counter;
    h.wait_own = l->wait_own, h.wait_lo = l->wait_lo, h.wait_hi = l->wait_hi, h.epoch = l->epoch;
  }
  return h;
}

__device__ __forceinline__ int ld_acquire_sys_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_acquire_gpu_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// consumer: one thread spins (bounded, ~10 s; the error word epoch[1] records a timeout)
__device__ __forceinline__ void halo_link_wait(const HaloLink& h) {
  if (!h.wait_own || !(h.wait_lo | h.wait_hi)) return;
  if (*(volatile const int*)(h.epoch + 1)) return;  // an earlier wait timed out: fail fast
  const int e = *(volatile const int*)h.epoch;
  const long long t0 = clock64();
  while ((h.wait_lo && ld_acquire_sys_i32(h.wait_own) < e) || (h.wait_hi && ld_acquire_sys_i32(h.wait_own + 1) < e)) {
    __nanosleep(128);
    if (clock64() - t0 > 20000000000LL) {
      atomicExch(const_cast<int*>(h.epoch) + 1, e);
      break;
    }
  }
}

// producer: called by thread 0 of every CTA after the CTA's last store (__syncthreads before).
// Every CTA fences at GPU scope and counts itself; the last one publishes with ONE
// system-scope fence (cumulative over the stores it observed through the counter).
__device__ __forceinline__ void halo_link_signal(const HaloLink& h) {
  if (!h.counter || !(h.lo || h.hi)) return;
  __threadfence();
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  if (atomicAdd(h.counter, 1u) == nblocks - 1) {
    *h.counter = 0;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const int e = *(volatile const int*)h.epoch;
    if (h.lo) asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(h.lo_flag), "r"(e) : "memory");
    if (h.hi) asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(h.hi_flag), "r"(e) : "memory");
  }
}

}  // namespace vm
