// box.cu — halo pack / unpack / unpack-add / zero-fill and dense<->slab layout
// kernels.  All HBM-bound copies: one 16-byte vector per thread where alignment
// allows, grid sized to a multiple of the SM count (grid-stride loops).
//
// Reference behaviour restated (bit-exact): halo.py:131-134 (send slabs are
// contiguous copies of the face), :139-148 (zero fill + concatenate),
// :176-186 (adjoint: receive and add); sharding.py:189-209 (block copies).
#include <cstdarg>
#include <atomic>
#include <cstdlib>

#include "vm_common.cuh"

namespace vm {

static thread_local char g_err[512];
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// per host thread: the threads mesh drives one rank per thread, each setting its own mode
static thread_local int g_pdl = -1;  // -1: from $VM_PDL (default off); 1: early trigger; 2: late (implicit) trigger
bool pdl_enabled() {
  if (g_pdl < 0) {
    const char* e = getenv("VM_PDL");
    g_pdl = (e && e[0] == '1') ? 1 : 0;
  }
  return g_pdl != 0;
}
bool pdl_late() { return pdl_enabled() && g_pdl == 2; }

static int g_num_sms = -1;
static int num_sms() {
  if (g_num_sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}
int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

struct Box {
  int64_t sd[5];   // strides of the big tensor in bytes
  int64_t lo[5];
  int64_t ext[5];  // ext[4] in units of `U` bytes after vectorisation
  int64_t rows;    // ext0*ext1*ext2*ext3
  int64_t units;   // per row
};

template <typename U>
__global__ void k_box_pack(const uint8_t* __restrict__ src, Box b, U* __restrict__ buf) {
  int64_t total = b.rows * b.units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = i % b.units, r = i / b.units;
    int64_t i3 = r % b.ext[3];
    r /= b.ext[3];
    int64_t i2 = r % b.ext[2];
    r /= b.ext[2];
    int64_t i1 = r % b.ext[1];
    int64_t i0 = r / b.ext[1];
    int64_t off = (b.lo[0] + i0) * b.sd[0] + (b.lo[1] + i1) * b.sd[1] + (b.lo[2] + i2) * b.sd[2] +
                  (b.lo[3] + i3) * b.sd[3] + b.lo[4] * b.sd[4] + u * (int64_t)sizeof(U);
    buf[i] = *reinterpret_cast<const U*>(src + off);
  }
}

template <typename U>
__global__ void k_box_unpack(uint8_t* __restrict__ dst, Box b, const U* __restrict__ buf) {
  int64_t total = b.rows * b.units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = i % b.units, r = i / b.units;
    int64_t i3 = r % b.ext[3];
    r /= b.ext[3];
    int64_t i2 = r % b.ext[2];
    r /= b.ext[2];
    int64_t i1 = r % b.ext[1];
    int64_t i0 = r / b.ext[1];
    int64_t off = (b.lo[0] + i0) * b.sd[0] + (b.lo[1] + i1) * b.sd[1] + (b.lo[2] + i2) * b.sd[2] +
                  (b.lo[3] + i3) * b.sd[3] + b.lo[4] * b.sd[4] + u * (int64_t)sizeof(U);
    *reinterpret_cast<U*>(dst + off) = buf ? buf[i] : U{};
  }
}

template <typename T>
__global__ void k_box_unpack_add(uint8_t* __restrict__ dst, Box b, const T* __restrict__ buf) {
  int64_t total = b.rows * b.units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = i % b.units, r = i / b.units;
    int64_t i3 = r % b.ext[3];
    r /= b.ext[3];
    int64_t i2 = r % b.ext[2];
    r /= b.ext[2];
    int64_t i1 = r % b.ext[1];
    int64_t i0 = r / b.ext[1];
    int64_t off = (b.lo[0] + i0) * b.sd[0] + (b.lo[1] + i1) * b.sd[1] + (b.lo[2] + i2) * b.sd[2] +
                  (b.lo[3] + i3) * b.sd[3] + b.lo[4] * b.sd[4] + u * (int64_t)sizeof(T);
    T* p = reinterpret_cast<T*>(dst + off);
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
      *p = __float2bfloat16_rn(__bfloat162float(*p) + __bfloat162float(buf[i]));
    } else {
      *p = *p + buf[i];
    }
  }
}

static int make_box(const int64_t dims[5], int eb, const int64_t lo[5], const int64_t ext[5],
                    Box& b, int& unit, const void* p1, const void* p2) {
  VM_REQUIRE(eb > 0, VM_E_ARG, "element size must be positive");
  for (int i = 0; i < 5; ++i) {
    VM_REQUIRE(dims[i] >= 0 && lo[i] >= 0 && ext[i] >= 0 && lo[i] + ext[i] <= dims[i], VM_E_SHAPE,
               "box [%lld,+%lld) outside dim %d of extent %lld", (long long)lo[i],
               (long long)ext[i], i, (long long)dims[i]);
  }
  int64_t st = eb;
  for (int i = 4; i >= 0; --i) {
    b.sd[i] = st;
    st *= dims[i];
  }
  int64_t rowbytes = ext[4] * eb;
  int64_t lobytes = lo[4] * eb;
  unit = 16;
  while (unit > 1 && (rowbytes % unit || lobytes % unit || b.sd[3] % unit ||
                      reinterpret_cast<uintptr_t>(p1) % unit ||
                      (p2 && reinterpret_cast<uintptr_t>(p2) % unit)))
    unit >>= 1;
  for (int i = 0; i < 5; ++i) {
    b.lo[i] = lo[i];
    b.ext[i] = ext[i];
  }
  b.rows = ext[0] * ext[1] * ext[2] * ext[3];
  b.units = rowbytes / unit;
  return VM_OK;
}

}  // namespace vm

using namespace vm;

extern "C" int vm_version(void) { return 1; }

extern "C" const char* vm_error_string(int code) {
  switch (code) {
    case VM_OK: return "ok";
    case VM_E_ARG: return "invalid argument";
    case VM_E_DTYPE: return "unsupported dtype";
    case VM_E_SHAPE: return "inconsistent shape";
    case VM_E_ALIGN: return "misaligned pointer or stride";
    case VM_E_HALO: return "halo margin exceeds local extent";
    case VM_E_UNSUPPORTED: return "unsupported configuration";
  }
  if (code > 0) return cudaGetErrorString(static_cast<cudaError_t>(code));
  return "unknown error";
}

extern "C" const char* vm_last_error(void) { return g_err; }

extern "C" long long vm_launch_count(void) { return g_launches.load(); }
extern "C" int vm_set_pdl(int on) {
  const int prev = vm::pdl_enabled() ? vm::g_pdl : 0;
  vm::g_pdl = on == 2 ? 2 : on ? 1 : 0;
  return prev;
}

extern "C" int vm_num_sms(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

#define BOX_LAUNCH(KERNEL, PTR, BUF, TYPEBUF)                                                \
  switch (unit) {                                                                            \
    case 16: KERNEL<int4><<<grid, 256, 0, st>>>(PTR, b, (TYPEBUF int4*)BUF); break;          \
    case 8: KERNEL<int2><<<grid, 256, 0, st>>>(PTR, b, (TYPEBUF int2*)BUF); break;           \
    case 4: KERNEL<int><<<grid, 256, 0, st>>>(PTR, b, (TYPEBUF int*)BUF); break;             \
    case 2: KERNEL<short><<<grid, 256, 0, st>>>(PTR, b, (TYPEBUF short*)BUF); break;         \
    default: KERNEL<char><<<grid, 256, 0, st>>>(PTR, b, (TYPEBUF char*)BUF); break;          \
  }

extern "C" int vm_box_pack(const void* src, const int64_t dims[5], int elem_bytes,
                           const int64_t lo[5], const int64_t ext[5], void* buf, void* stream) {
  VM_REQUIRE(src && buf && dims && lo && ext, VM_E_ARG, "vm_box_pack: null argument");
  Box b;
  int unit;
  int rc = make_box(dims, elem_bytes, lo, ext, b, unit, src, buf);
  if (rc) return rc;
  if (b.rows * b.units == 0) return VM_OK;
  cudaStream_t st = as_stream(stream);
  int grid = grid_for(b.rows * b.units, 256);
  const uint8_t* p = static_cast<const uint8_t*>(src);
  BOX_LAUNCH(k_box_pack, p, buf, )
  return launch_status("vm_box_pack");
}

extern "C" int vm_box_unpack(void* dst, const int64_t dims[5], int elem_bytes, const int64_t lo[5],
                             const int64_t ext[5], const void* buf, void* stream) {
  VM_REQUIRE(dst && buf && dims && lo && ext, VM_E_ARG, "vm_box_unpack: null argument");
  Box b;
  int unit;
  int rc = make_box(dims, elem_bytes, lo, ext, b, unit, dst, buf);
  if (rc) return rc;
  if (b.rows * b.units == 0) return VM_OK;
  cudaStream_t st = as_stream(stream);
  int grid = grid_for(b.rows * b.units, 256);
  uint8_t* p = static_cast<uint8_t*>(dst);
  BOX_LAUNCH(k_box_unpack, p, buf, const)
  return launch_status("vm_box_unpack");
}

extern "C" int vm_box_zero(void* dst, const int64_t dims[5], int elem_bytes, const int64_t lo[5],
                           const int64_t ext[5], void* stream) {
  VM_REQUIRE(dst && dims && lo && ext, VM_E_ARG, "vm_box_zero: null argument");
  Box b;
  int unit;
  int rc = make_box(dims, elem_bytes, lo, ext, b, unit, dst, nullptr);
  if (rc) return rc;
  if (b.rows * b.units == 0) return VM_OK;
  cudaStream_t st = as_stream(stream);
  int grid = grid_for(b.rows * b.units, 256);
  uint8_t* p = static_cast<uint8_t*>(dst);
  const void* nullbuf = nullptr;
  BOX_LAUNCH(k_box_unpack, p, nullbuf, const)
  return launch_status("vm_box_zero");
}

extern "C" int vm_box_unpack_add(void* dst, const int64_t dims[5], int dtype, const int64_t lo[5],
                                 const int64_t ext[5], const void* buf, void* stream) {
  VM_REQUIRE(dst && buf && dims && lo && ext, VM_E_ARG, "vm_box_unpack_add: null argument");
  int eb = dtype_bytes(dtype);
  VM_REQUIRE(dtype == VM_F32 || dtype == VM_F64 || dtype == VM_BF16, VM_E_DTYPE,
             "vm_box_unpack_add: dtype %d is not additive", dtype);
  Box b;
  int unit;
  int rc = make_box(dims, eb, lo, ext, b, unit, dst, buf);
  if (rc) return rc;
  // element-wise add: undo the vectorisation
  b.units = ext[4];
  if (b.rows * b.units == 0) return VM_OK;
  cudaStream_t st = as_stream(stream);
  int grid = grid_for(b.rows * b.units, 256);
  uint8_t* p = static_cast<uint8_t*>(dst);
  if (dtype == VM_F32)
    k_box_unpack_add<float><<<grid, 256, 0, st>>>(p, b, static_cast<const float*>(buf));
  else if (dtype == VM_F64)
    k_box_unpack_add<double><<<grid, 256, 0, st>>>(p, b, static_cast<const double*>(buf));
  else
    k_box_unpack_add<__nv_bfloat16><<<grid, 256, 0, st>>>(p, b, static_cast<const __nv_bfloat16*>(buf));
  return launch_status("vm_box_unpack_add");
}

// ------------------------------------------------------------------ dense <-> slab

template <typename S, typename T>
__global__ void k_dense_to_slab(const S* __restrict__ src, T* __restrict__ slab, Slab g, int B,
                                int C) {
  // one thread per (voxel, channel-block): writes one 8-channel vector
  int64_t nvox = (int64_t)B * g.D * g.H * g.W;
  int64_t total = nvox * g.CG;
  const bool fast = total < (1LL << 31) && g.mW;  // 32-bit multiply-high split (the usual case)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v;
    int cg, w, h, d, b;
    if (fast) {
      cg = (int)(i / nvox);  // nvox-sized runs: one 64-bit division per thread-iteration is fine here
      v = i - (int64_t)cg * nvox;
      const uint32_t v32 = (uint32_t)v;
      const uint32_t q1 = fastdiv(v32, (uint32_t)g.W, g.mW);
      w = (int)(v32 - q1 * (uint32_t)g.W);
      const uint32_t q2 = fastdiv(q1, (uint32_t)g.H, g.mH);
      h = (int)(q1 - q2 * (uint32_t)g.H);
      const uint32_t q3 = fastdiv(q2, (uint32_t)g.D, g.mD);
      d = (int)(q2 - q3 * (uint32_t)g.D);
      b = (int)q3;
    } else {
      v = i % nvox;
      cg = (int)(i / nvox);
      w = v % g.W;
      int64_t r = v / g.W;
      h = r % g.H;
      r /= g.H;
      d = r % g.D;
      b = (int)(r / g.D);
    }
    T out[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int c = cg * 8 + j;
      float val = c < C ? (float)src[v * C + c] : 0.f;
      out[j] = Cvt<T>::from_f(val);
    }
    T* dst = slab + g.at(b, cg, d, h, w);
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[j] = out[j];
  }
}

template <typename S, typename T>
__global__ void k_slab_to_dense(const S* __restrict__ slab, T* __restrict__ dst, Slab g, int B,
                                int C) {
  int64_t nvox = (int64_t)B * g.D * g.H * g.W;
  int64_t total = nvox * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = i % C;
    int64_t v = i / C;
    int w = v % g.W;
    int64_t r = v / g.W;
    int h = r % g.H;
    r /= g.H;
    int d = r % g.D;
    int b = (int)(r / g.D);
    float val = Cvt<S>::to_f(slab[g.at(b, c / 8, d, h, w) + (c % 8)]);
    dst[i] = (T)val;
  }
}

extern "C" int vm_dense_to_slab(const void* src, int src_dtype, void* slab, int slab_dtype,
                                int64_t bstride, int B, int C, int D, int H, int W, int m,
                                void* stream) {
  VM_REQUIRE(src && slab, VM_E_ARG, "vm_dense_to_slab: null pointer");
  VM_REQUIRE(B > 0 && C > 0 && D > 0 && H > 0 && W > 0 && m >= 0, VM_E_SHAPE,
             "vm_dense_to_slab: bad shape");
  VM_REQUIRE(src_dtype == VM_F32, VM_E_DTYPE, "vm_dense_to_slab: source must be f32");
  const Slab g = make_slab(bstride ? bstride : default_bstride(C, D, H, W, m), (C + 7) / 8, D, H, W, m);
  cudaStream_t st = as_stream(stream);
  int64_t work = (int64_t)B * D * H * W * g.CG;
  int grid = grid_for(work, 256);
  const float* s = static_cast<const float*>(src);
  if (slab_dtype == VM_BF16)
    k_dense_to_slab<float, __nv_bfloat16><<<grid, 256, 0, st>>>(s, (__nv_bfloat16*)slab, g, B, C);
  else if (slab_dtype == VM_F32)
    k_dense_to_slab<float, float><<<grid, 256, 0, st>>>(s, (float*)slab, g, B, C);
  else
    VM_REQUIRE(false, VM_E_DTYPE, "vm_dense_to_slab: slab dtype %d", slab_dtype);
  return launch_status("vm_dense_to_slab");
}

// Single-channel input in the compact padded layout [B][(D+2)(H+2)(W+2)] bf16 (zero margins):
// the operand of the Cin = 1 im2col convs (first_layer.cu), 2 bytes per voxel instead of the
// 16 of an 8-channel slab group.  One thread per padded row.
// one sample per grid row; 32-bit multiply-high (w, h) split (the 64-bit divisions of the
// first version ran this 12 MB conversion at ~16 us per e2e step)
__global__ void k_dense_to_compact1(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int D, int H,
                                    int W, uint32_t mWp, uint32_t mHp) {
  const uint32_t Hp = H + 2, Wp = W + 2;
  const uint32_t per = (uint32_t)(D + 2) * Hp * Wp;
  const int b = blockIdx.y;
  const float* sb = src + (int64_t)b * D * H * W;
  __nv_bfloat16* db = dst + (int64_t)b * per;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < per; r += gridDim.x * blockDim.x) {
    const uint32_t q = fastdiv(r, Wp, mWp);
    const int wq = (int)(r - q * Wp) - 1;
    const uint32_t dq1 = fastdiv(q, Hp, mHp);
    const int hq = (int)(q - dq1 * Hp) - 1;
    const int dq = (int)dq1 - 1;
    float v = 0.f;
    if (dq >= 0 && dq < D && hq >= 0 && hq < H && wq >= 0 && wq < W)
      v = sb[((int64_t)dq * H + hq) * W + wq];
    db[r] = __float2bfloat16_rn(v);
  }
}

extern "C" int vm_dense_to_compact1(const float* src, void* dst, int B, int D, int H, int W, void* stream) {
  VM_REQUIRE(src && dst && B > 0 && B < 65536, VM_E_ARG, "vm_dense_to_compact1: bad argument");
  const int64_t per = (int64_t)(D + 2) * (H + 2) * (W + 2);
  VM_REQUIRE(per < (1LL << 31) && H + 2 < 65536 && W + 2 < 65536, VM_E_SHAPE, "vm_dense_to_compact1: sample too large");
  int64_t gx = (per + 255) / 256;
  if (gx > 148 * 16) gx = 148 * 16;
  k_dense_to_compact1<<<dim3((unsigned)gx, (unsigned)B), 256, 0, as_stream(stream)>>>(
      src, (__nv_bfloat16*)dst, D, H, W, fastdiv_magic((uint32_t)(W + 2)), fastdiv_magic((uint32_t)(H + 2)));
  return launch_status("vm_dense_to_compact1");
}

extern "C" int vm_slab_to_dense(const void* slab, int slab_dtype, int64_t bstride, void* dst,
                                int dst_dtype, int B, int C, int D, int H, int W, int m,
                                void* stream) {
  VM_REQUIRE(slab && dst, VM_E_ARG, "vm_slab_to_dense: null pointer");
  VM_REQUIRE(dst_dtype == VM_F32, VM_E_DTYPE, "vm_slab_to_dense: destination must be f32");
  Slab g{bstride ? bstride : default_bstride(C, D, H, W, m), (C + 7) / 8, D, H, W, m};
  cudaStream_t st = as_stream(stream);
  int grid = grid_for((int64_t)B * D * H * W * C, 256);
  if (slab_dtype == VM_BF16)
    k_slab_to_dense<__nv_bfloat16, float><<<grid, 256, 0, st>>>((const __nv_bfloat16*)slab,
                                                               (float*)dst, g, B, C);
  else if (slab_dtype == VM_F32)
    k_slab_to_dense<float, float><<<grid, 256, 0, st>>>((const float*)slab, (float*)dst, g, B, C);
  else
    VM_REQUIRE(false, VM_E_DTYPE, "vm_slab_to_dense: slab dtype %d", slab_dtype);
  return launch_status("vm_slab_to_dense");
}

__global__ void k_onehot(const uint8_t* __restrict__ lab, float* __restrict__ oh, int64_t n,
                         int ncls) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * ncls;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = i % ncls;
    oh[i] = (lab[i / ncls] == c) ? 1.f : 0.f;
  }
}

// 3 classes: 4 voxels per thread, one 4-byte label load and three 16-byte stores (the scalar
// kernel above spends a 64-bit division per output float)
__global__ void k_onehot3x4(const uint8_t* __restrict__ lab, float* __restrict__ oh, int64_t n4) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t l4 = reinterpret_cast<const uint32_t*>(lab)[q];
    float o[12];
#pragma unroll
    for (int vv = 0; vv < 4; ++vv) {
      const uint32_t l = (l4 >> (8 * vv)) & 0xFFu;
#pragma unroll
      for (int c = 0; c < 3; ++c) o[vv * 3 + c] = l == (uint32_t)c ? 1.f : 0.f;
    }
    float4* dst = reinterpret_cast<float4*>(oh + q * 12);
    dst[0] = make_float4(o[0], o[1], o[2], o[3]);
    dst[1] = make_float4(o[4], o[5], o[6], o[7]);
    dst[2] = make_float4(o[8], o[9], o[10], o[11]);
  }
}

extern "C" int vm_onehot_u8(const uint8_t* labels, float* onehot, int64_t nvox, int ncls,
                            void* stream) {
  VM_REQUIRE(labels && onehot && nvox >= 0 && ncls > 0, VM_E_ARG, "vm_onehot_u8: bad argument");
  if (nvox == 0) return VM_OK;
  if (ncls == 3 && nvox % 4 == 0 && (reinterpret_cast<uintptr_t>(labels) & 3) == 0 &&
      (reinterpret_cast<uintptr_t>(onehot) & 15) == 0) {
    k_onehot3x4<<<grid_for(nvox / 4, 256), 256, 0, as_stream(stream)>>>(labels, onehot, nvox / 4);
    return launch_status("vm_onehot_u8");
  }
  k_onehot<<<grid_for(nvox * ncls, 256), 256, 0, as_stream(stream)>>>(labels, onehot, nvox, ncls);
  return launch_status("vm_onehot_u8");
}
