// halo.cu — the halo exchange of a channel-blocked padded slab as ONE stream-ordered C call
// (SURVEY §8(b) vm_halo_fwd), plus the weight-gradient / statistics all-reduce
// (vm_allreduce_f32), over the caller's NCCL communicator.
//
// Protocol (halo.py:109-155, restated): the three spatial dims are exchanged one after the
// other (D, then H, then W); the face sent in phase a spans the margins filled by phases < a,
// so edges and corners arrive over 2-3 hops with no diagonal messages, and the bytes equal
// halo.exchange_byte_count (halo.py:197-229).  Margin 1 (k = 3).  Per phase:
//   pack    one launch: the first interior layer ("down", to the lo neighbour) and the last
//           ("up", to the hi neighbour) of every (sample, channel group) into two contiguous
//           messages [B][CG][n1][n2][8];
//   NCCL    one group: send up, send down, recv from lo, recv from hi (per-peer issue order
//           makes a rank that is its own lo AND hi neighbour — the periodic single-GPU
//           emulation — receive the up message in its lo margin, as a ring would);
//   unpack  one launch into margin layer 0 (from lo) and n+1 (from hi).
// Global-boundary margins are never written: they stay zero from allocation (halo.py:136-147).
//
// NCCL is not linked: the entry points bind ncclSend/ncclRecv/ncclGroupStart/ncclGroupEnd/
// ncclAllReduce from the libnccl.so.2 already loaded by the process (torch's), so the
// communicator the caller passes (ProcessGroupNCCL._comm_ptr()) and these calls are the same
// NCCL instance.  All work is enqueued on the caller's stream (capturable in a CUDA graph).
#include <cuda.h>
#include <dlfcn.h>

#include <cstring>

#include "vm_common.cuh"

namespace vm {

// ------------------------------------------------------------------ face kernels
// A face: the layer `pos` (padded index) along `axis` of every (sample, channel group), over
// the padded extents of the dims exchanged before `axis` and the interior of those after it
// (full = 1: the whole padded cross-section, used by vm_halo_slab_zero).
struct Face {
  int axis, pos, full;
  uint8_t* buf;  // message [B][CG][n1][n2][vec] (nullptr on unpack: zero fill)
};
struct FaceSet {
  Face f[6];
  int n;
  int64_t bstride_b, plane_b;  // bytes
  int CG, B, D, H, W;
  int vec;  // bytes per voxel-group (8 channels)
};

__host__ __device__ inline void face_extent(const FaceSet& s, const Face& f, int& n1, int& n2, int& lo1, int& lo2) {
  const int Dp = s.D + 2, Hp = s.H + 2;
  if (f.axis == 0) {  // (h, w)
    n1 = f.full ? Hp : s.H, n2 = f.full ? s.W + 2 : s.W, lo1 = f.full ? 0 : 1, lo2 = f.full ? 0 : 1;
  } else if (f.axis == 1) {  // (d, w): d padded (phase 0 came first)
    n1 = Dp, n2 = f.full ? s.W + 2 : s.W, lo1 = 0, lo2 = f.full ? 0 : 1;
  } else {  // (d, h), both padded
    n1 = Dp, n2 = Hp, lo1 = 0, lo2 = 0;
  }
}

// One warp per row of a face: a row is the run along the face's last dim (i2) of one
// (sample, channel group, i1); lanes stride over its 16-byte units (a whole W row of a depth
// or height face is contiguous in the slab: 512-byte warp accesses).  32-bit index math.
template <bool PACK>
__global__ void __launch_bounds__(256) k_slab_faces(uint8_t* __restrict__ slab, const FaceSet s) {
  pdl_wait();
  const Face f = s.f[blockIdx.y];
  int n1, n2, lo1, lo2;
  face_extent(s, f, n1, n2, lo1, lo2);
  const int upv = s.vec / 16;  // 16-byte units per voxel group (1: bf16, 2: f32)
  const int rows = s.B * s.CG * n1;
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  if (row >= rows) return;
  const int lane = threadIdx.x % 32;
  const int i1 = row % n1;
  const int bc = row / n1;
  const int cg = bc % s.CG, b = bc / s.CG;
  const int Hp = s.H + 2, Wp = s.W + 2;
  // slab byte offset of (i1, i2 = 0) and the byte stride along i2
  int64_t base;
  int64_t step;
  if (f.axis == 0) base = ((int64_t)f.pos * Hp + lo1 + i1) * Wp + lo2, step = 1;
  else if (f.axis == 1) base = ((int64_t)(lo1 + i1) * Hp + f.pos) * Wp + lo2, step = 1;
  else base = ((int64_t)(lo1 + i1) * Hp + lo2) * Wp + f.pos, step = Wp;
  uint8_t* p0 = slab + b * s.bstride_b + cg * s.plane_b + base * s.vec;
  const int units = n2 * upv;
  uint4* msg = f.buf ? reinterpret_cast<uint4*>(f.buf) + (int64_t)row * units : nullptr;
  for (int u = lane; u < units; u += 32) {
    const int i2 = u / upv, k = u - i2 * upv;
    uint4* p = reinterpret_cast<uint4*>(p0 + (int64_t)i2 * step * s.vec) + k;
    if (PACK) msg[u] = *p;
    else *p = msg ? msg[u] : make_uint4(0, 0, 0, 0);
  }
}

static int64_t face_bytes(const FaceSet& s, const Face& f) {
  int n1, n2, lo1, lo2;
  face_extent(s, f, n1, n2, lo1, lo2);
  return (int64_t)s.B * s.CG * n1 * n2 * s.vec;
}

static int launch_faces(bool pack, void* slab, const FaceSet& s, cudaStream_t st) {
  if (s.n == 0) return VM_OK;
  int most = 0;
  for (int i = 0; i < s.n; ++i) {
    int n1, n2, lo1, lo2;
    face_extent(s, s.f[i], n1, n2, lo1, lo2);
    const int rows = s.B * s.CG * n1;
    most = rows > most ? rows : most;
  }
  dim3 grid((most + 7) / 8, s.n);
  if (pack) launch_pdl(k_slab_faces<true>, grid, 256, 0, st, static_cast<uint8_t*>(slab), s);
  else launch_pdl(k_slab_faces<false>, grid, 256, 0, st, static_cast<uint8_t*>(slab), s);
  return launch_status(pack ? "vm_halo pack" : "vm_halo unpack");
}

static FaceSet face_set(int dtype, int64_t bstride, int B, int C, int D, int H, int W) {
  FaceSet s{};
  const int eb = dtype_bytes(dtype);
  s.vec = 8 * eb;
  s.CG = (C + 7) / 8;
  s.B = B, s.D = D, s.H = H, s.W = W;
  s.plane_b = (int64_t)(D + 2) * (H + 2) * (W + 2) * s.vec;
  s.bstride_b = (bstride ? bstride : (int64_t)s.CG * (D + 2) * (H + 2) * (W + 2) * 8) * eb;
  return s;
}

// ------------------------------------------------------------------ NCCL, bound at run time
typedef int (*nccl_p2p_t)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_t)();
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_t)(int);
struct NcclApi {
  nccl_p2p_t send = nullptr, recv = nullptr;
  nccl_group_t gstart = nullptr, gend = nullptr;
  nccl_allreduce_t allreduce = nullptr;
  nccl_errstr_t errstr = nullptr;
};
static NcclApi g_nccl;
constexpr int kNcclUint8 = 1, kNcclFloat32 = 7, kNcclSum = 0;  // ncclDataType_t / ncclRedOp_t values

// smallest padded layer (bytes per sample and channel group) sent without packing
// (vm_set_halo_zero_copy_min).  Off by default: measured on B200 (tools/halo_ab.py, cfg3
// 8-way rank block), one NCCL op per channel group cost more than the pack + one message +
// unpack (sum of the forward exchanges 1961 us zero-copy vs 909 us packed)
static long long g_zero_copy_min = 1LL << 62;
extern "C" long long vm_set_halo_zero_copy_min(long long bytes) {
  const long long prev = g_zero_copy_min;
  g_zero_copy_min = bytes;
  return prev;
}

static int g_loopback = 0;
extern "C" void vm_debug_halo_loopback(int on) { g_loopback = on; }

static bool nccl_ok() { return g_nccl.send && g_nccl.recv && g_nccl.gstart && g_nccl.gend && g_nccl.allreduce; }

#define NCCL_CHECK(call, what)                                                              \
  do {                                                                                      \
    const int _r = (call);                                                                  \
    if (_r != 0) {                                                                          \
      set_error("%s: NCCL error %d (%s)", what, _r, g_nccl.errstr ? g_nccl.errstr(_r) : "?"); \
      return 1000 + _r;                                                                     \
    }                                                                                       \
  } while (0)

}  // namespace vm

using namespace vm;

extern "C" int vm_nccl_bind(void) {
  if (nccl_ok()) return VM_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch's)
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  VM_REQUIRE(h, VM_E_UNSUPPORTED, "vm_nccl_bind: libnccl.so.2 not loadable (%s)", dlerror());
  g_nccl.send = reinterpret_cast<nccl_p2p_t>(dlsym(h, "ncclSend"));
  g_nccl.recv = reinterpret_cast<nccl_p2p_t>(dlsym(h, "ncclRecv"));
  g_nccl.gstart = reinterpret_cast<nccl_group_t>(dlsym(h, "ncclGroupStart"));
  g_nccl.gend = reinterpret_cast<nccl_group_t>(dlsym(h, "ncclGroupEnd"));
  g_nccl.allreduce = reinterpret_cast<nccl_allreduce_t>(dlsym(h, "ncclAllReduce"));
  g_nccl.errstr = reinterpret_cast<nccl_errstr_t>(dlsym(h, "ncclGetErrorString"));
  VM_REQUIRE(nccl_ok(), VM_E_UNSUPPORTED, "vm_nccl_bind: NCCL symbols missing");
  return VM_OK;
}

extern "C" size_t vm_halo_slab_ws_bytes(int dtype, int B, int C, int D, int H, int W) {
  FaceSet s = face_set(dtype, 0, B, C, D, H, W);
  int64_t most = 0;
  for (int a = 0; a < 3; ++a) {
    Face f{a, 1, 0, nullptr};
    const int64_t b = face_bytes(s, f);
    most = b > most ? b : most;
  }
  return (size_t)(4 * ((most + 255) / 256 * 256));  // 2 send + 2 recv messages
}

// Forward halo of a slab (halo.py:109-155).  nbr[2a] / nbr[2a+1] = lo / hi neighbour rank of
// spatial dim a (D, H, W) in the communicator, -1 at a global boundary.  ws: device scratch of
// vm_halo_slab_ws_bytes.  bytes_sent (optional, host) accumulates the message bytes.
extern "C" int vm_halo_slab_fwd(void* comm, int dtype, void* slab, int64_t bstride, int B, int C, int D, int H,
                                int W, const int* nbr, void* ws, size_t ws_bytes, long long* bytes_sent,
                                void* stream) {
  VM_REQUIRE(slab && nbr && ws, VM_E_ARG, "vm_halo_slab_fwd: null pointer");
  VM_REQUIRE(dtype == VM_BF16 || dtype == VM_F32, VM_E_UNSUPPORTED, "vm_halo_slab_fwd: dtype %d", dtype);
  VM_REQUIRE(D >= 1 && H >= 1 && W >= 1, VM_E_HALO, "vm_halo_slab_fwd: margin 1 exceeds local extent (%d,%d,%d)",
             D, H, W);
  VM_REQUIRE(ws_bytes >= vm_halo_slab_ws_bytes(dtype, B, C, D, H, W), VM_E_ARG, "vm_halo_slab_fwd: ws too small");
  VM_REQUIRE((reinterpret_cast<uintptr_t>(slab) & 15) == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0,
             VM_E_ALIGN, "vm_halo_slab_fwd: 16-byte alignment required");
  cudaStream_t st = as_stream(stream);
  const FaceSet base = face_set(dtype, bstride, B, C, D, H, W);
  const int n[3] = {D, H, W};
  const size_t quarter = ws_bytes / 4 / 256 * 256;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  uint8_t *s_down = w8, *s_up = w8 + quarter, *r_lo = w8 + 2 * quarter, *r_hi = w8 + 3 * quarter;
  for (int a = 0; a < 3; ++a) {
    const int lo = nbr[2 * a], hi = nbr[2 * a + 1];
    if (lo < 0 && hi < 0) continue;
    VM_REQUIRE(comm, VM_E_ARG, "vm_halo_slab_fwd: neighbours given without a communicator");
    VM_REQUIRE(nccl_ok() || vm_nccl_bind() == VM_OK, VM_E_UNSUPPORTED, "vm_halo_slab_fwd: NCCL not bound");
    if (a == 0 && base.plane_b / (D + 2) >= g_zero_copy_min) {
      // Depth phase, zero copy: every (sample, channel group)'s padded layer is one contiguous
      // run, sent from layer 1 / D and received straight into margin layer 0 / D+1.  The layer's
      // own H/W margins travel too: at a global boundary they are zero on both ranks, and on a
      // side with a neighbour the later H / W phases overwrite them (their boxes span the
      // depth margins), so the slab ends up identical to the packed protocol's; the bytes
      // exceed exchange_byte_count's face by (H+2)(W+2)/(HW).
      const size_t lb = (size_t)(base.plane_b / (D + 2));
      uint8_t* s8 = static_cast<uint8_t*>(slab);
      NCCL_CHECK(g_nccl.gstart(), "ncclGroupStart");
      for (int b = 0; b < B; ++b)
        for (int cg = 0; cg < base.CG; ++cg) {
          uint8_t* p = s8 + b * base.bstride_b + cg * base.plane_b;
          if (hi >= 0) NCCL_CHECK(g_nccl.send(p + (size_t)D * lb, lb, kNcclUint8, hi, comm, st), "ncclSend");
          if (lo >= 0) NCCL_CHECK(g_nccl.send(p + lb, lb, kNcclUint8, lo, comm, st), "ncclSend");
          if (lo >= 0) NCCL_CHECK(g_nccl.recv(p, lb, kNcclUint8, lo, comm, st), "ncclRecv");
          if (hi >= 0) NCCL_CHECK(g_nccl.recv(p + (size_t)(D + 1) * lb, lb, kNcclUint8, hi, comm, st), "ncclRecv");
        }
      NCCL_CHECK(g_nccl.gend(), "ncclGroupEnd");
      if (bytes_sent) *bytes_sent += (long long)lb * B * base.CG * ((lo >= 0) + (hi >= 0));
      continue;
    }
    FaceSet pk = base, up = base;
    pk.n = up.n = 0;
    if (lo >= 0) pk.f[pk.n++] = Face{a, 1, 0, s_down};
    if (hi >= 0) pk.f[pk.n++] = Face{a, n[a], 0, s_up};
    const size_t bytes = (size_t)face_bytes(base, Face{a, 1, 0, nullptr});
    int rc = launch_faces(true, slab, pk, st);
    if (rc) return rc;
    if (g_loopback) {  // A/B probe: the periodic self-exchange as device copies instead of NCCL
      if (lo >= 0 && hi >= 0) {
        cudaMemcpyAsync(r_lo, s_up, bytes, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(r_hi, s_down, bytes, cudaMemcpyDeviceToDevice, st);
      }
    } else {
    NCCL_CHECK(g_nccl.gstart(), "ncclGroupStart");
    if (hi >= 0) NCCL_CHECK(g_nccl.send(s_up, bytes, kNcclUint8, hi, comm, st), "ncclSend");
    if (lo >= 0) NCCL_CHECK(g_nccl.send(s_down, bytes, kNcclUint8, lo, comm, st), "ncclSend");
    if (lo >= 0) NCCL_CHECK(g_nccl.recv(r_lo, bytes, kNcclUint8, lo, comm, st), "ncclRecv");
    if (hi >= 0) NCCL_CHECK(g_nccl.recv(r_hi, bytes, kNcclUint8, hi, comm, st), "ncclRecv");
    NCCL_CHECK(g_nccl.gend(), "ncclGroupEnd");
    }
    if (lo >= 0) up.f[up.n++] = Face{a, 0, 0, r_lo};
    if (hi >= 0) up.f[up.n++] = Face{a, n[a] + 1, 0, r_hi};
    rc = launch_faces(false, slab, up, st);
    if (rc) return rc;
    if (bytes_sent) *bytes_sent += (long long)bytes * ((lo >= 0) + (hi >= 0));
  }
  return VM_OK;
}

// Zero the margin layers a halo wrote (sides with a neighbour), full padded cross-sections:
// the weight gradient reads a gradient slab's margins as zeros.  One launch.
extern "C" int vm_halo_slab_zero(int dtype, void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                                 const int* nbr, void* stream) {
  VM_REQUIRE(slab && nbr, VM_E_ARG, "vm_halo_slab_zero: null pointer");
  FaceSet s = face_set(dtype, bstride, B, C, D, H, W);
  const int n[3] = {D, H, W};
  s.n = 0;
  for (int a = 0; a < 3; ++a) {
    if (nbr[2 * a] >= 0) s.f[s.n++] = Face{a, 0, 1, nullptr};
    if (nbr[2 * a + 1] >= 0) s.f[s.n++] = Face{a, n[a] + 1, 1, nullptr};
  }
  return launch_faces(false, slab, s, as_stream(stream));
}

// Single-phase building blocks (the host-driven transports of the threads / gloo meshes use
// these around their own send/recv): pack the down/up messages of phase `axis`, or unpack the
// lo/hi messages into its margins.  A null message pointer skips that side.
extern "C" int vm_halo_slab_pack(int dtype, const void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                                 int axis, void* down, void* up, void* stream) {
  VM_REQUIRE(slab && axis >= 0 && axis < 3, VM_E_ARG, "vm_halo_slab_pack: bad argument");
  FaceSet s = face_set(dtype, bstride, B, C, D, H, W);
  const int n[3] = {D, H, W};
  s.n = 0;
  if (down) s.f[s.n++] = Face{axis, 1, 0, static_cast<uint8_t*>(down)};
  if (up) s.f[s.n++] = Face{axis, n[axis], 0, static_cast<uint8_t*>(up)};
  return launch_faces(true, const_cast<void*>(slab), s, as_stream(stream));
}
extern "C" int vm_halo_slab_unpack(int dtype, void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                                   int axis, const void* from_lo, const void* from_hi, void* stream) {
  VM_REQUIRE(slab && axis >= 0 && axis < 3, VM_E_ARG, "vm_halo_slab_unpack: bad argument");
  FaceSet s = face_set(dtype, bstride, B, C, D, H, W);
  const int n[3] = {D, H, W};
  s.n = 0;
  if (from_lo) s.f[s.n++] = Face{axis, 0, 0, static_cast<uint8_t*>(const_cast<void*>(from_lo))};
  if (from_hi) s.f[s.n++] = Face{axis, n[axis] + 1, 0, static_cast<uint8_t*>(const_cast<void*>(from_hi))};
  return launch_faces(false, slab, s, as_stream(stream));
}
extern "C" long long vm_halo_slab_face_bytes(int dtype, int B, int C, int D, int H, int W, int axis) {
  FaceSet s = face_set(dtype, 0, B, C, D, H, W);
  return face_bytes(s, Face{axis, 1, 0, nullptr});
}

// ------------------------------------------------------------------ one-phase halo (3-D meshes)
// The same margins as the 3-phase protocol in ONE round: every rank sends its boundary boxes
// straight to all (up to 26) face, edge and corner neighbours.  Direction k = index of the
// offset s = (sd, sh, sw) in {-1,0,1}^3 \ {0}, lexicographic (opp(k) = 25 - k).  The message
// for direction s is the interior box at layer 1 (s = -1) / n (s = +1) / 1..n (s = 0) per
// axis; the message from the neighbour at offset s lands in the margin box at layer 0 / n+1 /
// 1..n.  A corner or edge value is the diagonal neighbour's own interior voxel either way, so
// the slab is byte-identical to the sequential protocol's (halo.py:109-155, where it travels
// over 2-3 hops); at a global boundary nothing is sent and the margin stays zero.  Per
// exchange: one pack launch, one NCCL group, one unpack launch (the 3-phase path: 3 of each).
// Issue order: sends for k ascending; receives for k ascending from the neighbour at offset
// opp(k) — so for every pair of ranks both sides walk their common directions in the same
// order, and a rank that is every neighbour of itself (the periodic single-GPU emulation)
// receives the message of direction k in its margin on side opp(k), as a torus would.
struct Box {
  int lo[3], n[3];
  uint8_t* buf;
};
struct BoxSet {
  Box b[26];
  int start[27];  // prefix sums of the boxes' 16-byte units (one flat grid over all boxes)
  int n;
  int64_t bstride_b, plane_b;
  int CG, B, D, H, W;
  int vec;
};

__host__ __device__ inline int64_t box_units(const BoxSet& s, const Box& x) {
  return (int64_t)s.B * s.CG * x.n[0] * x.n[1] * x.n[2] * (s.vec / 16);
}

template <bool PACK>
__global__ void __launch_bounds__(256) k_slab_boxes(uint8_t* __restrict__ slab, const BoxSet s) {
  pdl_wait();
  const int upv = s.vec / 16;
  const int Hp = s.H + 2, Wp = s.W + 2;
  const int total = s.start[s.n];
  // one flat grid over all boxes (26 per-box grids left ~20 us of empty blocks at 256^3);
  // consecutive threads walk a box's last dim (a contiguous run of the slab when it is W)
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    int j = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1)  // largest j with start[j] <= g
      if (j + step < s.n && s.start[j + step] <= g) j += step;
    const Box& x = s.b[j];
    const int u = g - s.start[j];
    const int n2u = x.n[2] * upv;
    const int r = u / n2u, w = u - r * n2u;  // (b, cg, i0, i1) row, unit within the row
    const int i1 = r % x.n[1], r2 = r / x.n[1];
    const int i0 = r2 % x.n[0], bc = r2 / x.n[0];
    const int cg = bc % s.CG, b = bc / s.CG;
    const int64_t row = ((int64_t)(x.lo[0] + i0) * Hp + x.lo[1] + i1) * Wp + x.lo[2];
    uint4* p = reinterpret_cast<uint4*>(slab + b * s.bstride_b + cg * s.plane_b + row * s.vec) + w;
    uint4* m = reinterpret_cast<uint4*>(x.buf) + u;
    if (PACK) *m = *p;
    else *p = *m;
  }
}

static int launch_boxes(bool pack, void* slab, BoxSet& s, cudaStream_t st) {
  if (s.n == 0) return VM_OK;
  s.start[0] = 0;
  for (int i = 0; i < s.n; ++i) s.start[i + 1] = s.start[i] + (int)box_units(s, s.b[i]);
  int64_t gx = ((int64_t)s.start[s.n] + 255) / 256;
  if (gx > 148 * 8) gx = 148 * 8;  // grid-stride beyond one full wave
  if (pack) launch_pdl(k_slab_boxes<true>, dim3((unsigned)gx), 256, 0, st, static_cast<uint8_t*>(slab), s);
  else launch_pdl(k_slab_boxes<false>, dim3((unsigned)gx), 256, 0, st, static_cast<uint8_t*>(slab), s);
  return launch_status(pack ? "vm_halo26 pack" : "vm_halo26 unpack");
}

// box of direction k: send (interior boundary) or recv (margin on side s)
static Box dir_box(int k, bool recv, int D, int H, int W) {
  const int t = k < 13 ? k : k + 1;
  const int s[3] = {t / 9 - 1, (t / 3) % 3 - 1, t % 3 - 1};
  const int n[3] = {D, H, W};
  Box x{};
  for (int a = 0; a < 3; ++a) {
    x.n[a] = s[a] == 0 ? n[a] : 1;
    x.lo[a] = s[a] == 0 ? 1 : (s[a] < 0 ? (recv ? 0 : 1) : (recv ? n[a] + 1 : n[a]));
  }
  return x;
}

static int64_t box_bytes(const BoxSet& s, const Box& x) { return box_units(s, x) * 16; }

extern "C" size_t vm_halo_slab_ws_bytes26(int dtype, int B, int C, int D, int H, int W) {
  BoxSet s{};
  const FaceSet f = face_set(dtype, 0, B, C, D, H, W);
  s.vec = f.vec, s.CG = f.CG, s.B = B;
  size_t tot = 0;
  for (int k = 0; k < 26; ++k) tot += (size_t)((box_bytes(s, dir_box(k, false, D, H, W)) + 255) / 256 * 256);
  return 2 * tot;
}

extern "C" int vm_halo_slab_fwd26(void* comm, int dtype, void* slab, int64_t bstride, int B, int C, int D, int H,
                                  int W, const int* nbr26, void* ws, size_t ws_bytes, long long* bytes_sent,
                                  void* stream) {
  VM_REQUIRE(slab && nbr26 && ws, VM_E_ARG, "vm_halo_slab_fwd26: null pointer");
  VM_REQUIRE(dtype == VM_BF16 || dtype == VM_F32, VM_E_UNSUPPORTED, "vm_halo_slab_fwd26: dtype %d", dtype);
  VM_REQUIRE(D >= 1 && H >= 1 && W >= 1, VM_E_HALO, "vm_halo_slab_fwd26: margin 1 exceeds local extent (%d,%d,%d)",
             D, H, W);
  VM_REQUIRE(ws_bytes >= vm_halo_slab_ws_bytes26(dtype, B, C, D, H, W), VM_E_ARG, "vm_halo_slab_fwd26: ws too small");
  VM_REQUIRE((reinterpret_cast<uintptr_t>(slab) & 15) == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0,
             VM_E_ALIGN, "vm_halo_slab_fwd26: 16-byte alignment required");
  int any = 0;
  for (int k = 0; k < 26; ++k) any |= nbr26[k] >= 0;
  if (!any) return VM_OK;
  VM_REQUIRE(comm, VM_E_ARG, "vm_halo_slab_fwd26: neighbours given without a communicator");
  VM_REQUIRE(nccl_ok() || vm_nccl_bind() == VM_OK, VM_E_UNSUPPORTED, "vm_halo_slab_fwd26: NCCL not bound");
  cudaStream_t st = as_stream(stream);
  const FaceSet f = face_set(dtype, bstride, B, C, D, H, W);
  BoxSet snd{}, rcv{};
  snd.bstride_b = rcv.bstride_b = f.bstride_b, snd.plane_b = rcv.plane_b = f.plane_b;
  snd.CG = rcv.CG = f.CG, snd.B = rcv.B = B, snd.D = rcv.D = D, snd.H = rcv.H = H, snd.W = rcv.W = W;
  snd.vec = rcv.vec = f.vec;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  const size_t half = vm_halo_slab_ws_bytes26(dtype, B, C, D, H, W) / 2;
  uint8_t* sp = w8;
  uint8_t* rp = w8 + half;
  uint8_t* sbuf[26] = {};
  uint8_t* rbuf[26] = {};
  size_t nbytes[26] = {};
  for (int k = 0; k < 26; ++k) {
    Box x = dir_box(k, false, D, H, W);
    nbytes[k] = (size_t)box_bytes(snd, x);
    const size_t adv = (nbytes[k] + 255) / 256 * 256;
    sbuf[k] = sp, rbuf[k] = rp;  // the slot of direction k in both halves
    sp += adv, rp += adv;
    if (nbr26[k] >= 0) {
      x.buf = sbuf[k];
      snd.b[snd.n++] = x;
    }
  }
  int rc = launch_boxes(true, slab, snd, st);
  if (rc) return rc;
  long long sent = 0;
  for (int k = 0; k < 26; ++k) sent += nbr26[k] >= 0 ? (long long)nbytes[k] : 0;
  if (g_loopback) {  // A/B probe: the periodic self-exchange as one device copy (no NCCL)
    cudaMemcpyAsync(rbuf[0], sbuf[0], half, cudaMemcpyDeviceToDevice, st);
  } else {
    // a run of consecutive directions with the same peer is one message (its slots are
    // contiguous in ws, in k order, on both sides: the receiver's run from that rank covers
    // the same k) — one NCCL op per neighbour on a 2x2x2 mesh, one in all for the emulation
    NCCL_CHECK(g_nccl.gstart(), "ncclGroupStart");
    for (int k = 0; k < 26;) {
      int e = k + 1;
      if (nbr26[k] >= 0) {
        while (e < 26 && nbr26[e] == nbr26[k]) ++e;
        NCCL_CHECK(g_nccl.send(sbuf[k], (size_t)(sbuf[e - 1] - sbuf[k]) + nbytes[e - 1], kNcclUint8, nbr26[k], comm,
                               st), "ncclSend");
      }
      k = e;
    }
    for (int k = 0; k < 26;) {
      const int from = nbr26[25 - k];  // the neighbour at offset opp(k) sent its direction-k box
      int e = k + 1;
      if (from >= 0) {
        while (e < 26 && nbr26[25 - e] == from) ++e;
        NCCL_CHECK(g_nccl.recv(rbuf[k], (size_t)(rbuf[e - 1] - rbuf[k]) + nbytes[e - 1], kNcclUint8, from, comm, st),
                   "ncclRecv");
      }
      k = e;
    }
    NCCL_CHECK(g_nccl.gend(), "ncclGroupEnd");
  }
  for (int k = 0; k < 26; ++k)
    if (nbr26[25 - k] >= 0) {
      Box x = dir_box(25 - k, true, D, H, W);  // margin on the side of the sender (offset opp(k))
      x.buf = rbuf[k];
      rcv.b[rcv.n++] = x;
    }
  rc = launch_boxes(false, slab, rcv, st);
  if (rc) return rc;
  if (bytes_sent) *bytes_sent += sent;
  return VM_OK;
}

// In-place sum of n floats over the communicator (the weight-gradient / loss-statistics
// all-reduce, mesh.py:195-233 / unet.py:434-441), on the caller's stream.
extern "C" int vm_allreduce_f32(void* comm, float* buf, size_t n, void* stream) {
  VM_REQUIRE(comm && buf, VM_E_ARG, "vm_allreduce_f32: null pointer");
  VM_REQUIRE(nccl_ok() || vm_nccl_bind() == VM_OK, VM_E_UNSUPPORTED, "vm_allreduce_f32: NCCL not bound");
  if (n == 0) return VM_OK;
  NCCL_CHECK(g_nccl.allreduce(buf, buf, n, kNcclFloat32, kNcclSum, comm, as_stream(stream)), "ncclAllReduce");
  return VM_OK;
}

// ------------------------------------------------------------------ peer-memory depth halo
// The depth phase of a depth-only split without NCCL: every rank PUSHES its first and last
// interior layers straight into its neighbours' margin layers through mapped peer memory
// (NVLink P2P stores; CUDA-IPC mappings of the neighbours' slabs), then signals them, then
// waits for its own margins.  One launch per exchange, no pack / unpack pass: a depth layer of
// a (sample, channel group) is one contiguous run of (H+2)(W+2) voxel groups, so the push is a
// flat 16-byte copy.  The whole padded layer moves; its H / W margins are zero on every rank
// of a depth-only split, so the slab ends up byte-identical to the packed protocol's
// (halo.py:109-155 with only `x` partitioned).
//
// Completion: every block fences its stores system-wide and counts itself done; the last
// block writes the step's epoch into the neighbours' flag words (release, system scope) and
// spins until its own two flag words (written by the neighbours' pushes) reach the epoch.  A
// rank that is its own neighbour (the periodic single-GPU emulation) signals itself before it
// waits, so it never waits on another kernel.
namespace vm {
struct DepthPush {
  const uint8_t* src;
  uint8_t* lo_dst;  // lo neighbour's slab (receives our layer 1 in its layer D+1), or null
  uint8_t* hi_dst;  // hi neighbour's slab (receives our layer D in its layer 0), or null
  int* lo_flag;     // the lo neighbour's "from hi" flag word
  int* hi_flag;     // the hi neighbour's "from lo" flag word
  int* own;         // own flag words [from lo, from hi]
  unsigned* counter;
  const int* epoch;
  int64_t bstride_b, plane_b, layer_b;
  int B, CG, D, wait_lo, wait_hi;
};

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(int* p, int v) {
  asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid: x over the 16-byte units of one layer, y over (sample, channel group, side).  Every
// block fences its stores at GPU scope and counts itself done; the last block (which has
// observed every other block's count, so their stores precede it in causality order) issues
// the one system-scope fence and the release stores that the neighbours acquire.
__device__ int g_push_dbg;  // A/B probe bits (vm_debug_push_mode): 1 gpu-scope publish, 2 no wait
__global__ void __launch_bounds__(256) k_depth_push(const DepthPush p) {
  pdl_wait();
  const unsigned n16 = (unsigned)(p.layer_b / 16);  // 16-byte units per layer
  const int sides = (p.lo_dst != nullptr) + (p.hi_dst != nullptr);
  const int r = blockIdx.y;
  const int s = r % sides;
  const int bc = r / sides;
  const int cg = bc % p.CG, b = bc / p.CG;
  const bool lo = s == 0 && p.lo_dst != nullptr;
  const int64_t base = b * p.bstride_b + cg * p.plane_b;
  const uint4* from = reinterpret_cast<const uint4*>(p.src + base + (lo ? 1 : p.D) * p.layer_b);
  uint4* to = reinterpret_cast<uint4*>((lo ? p.lo_dst : p.hi_dst) + base + (lo ? p.D + 1 : 0) * p.layer_b);
  const unsigned step = gridDim.x * blockDim.x;
  unsigned u = blockIdx.x * blockDim.x + threadIdx.x;
  for (; u + 3 * step < n16; u += 4 * step) {  // 4 loads in flight per thread
    const uint4 a0 = __ldg(from + u), a1 = __ldg(from + u + step), a2 = __ldg(from + u + 2 * step),
                a3 = __ldg(from + u + 3 * step);
    to[u] = a0, to[u + step] = a1, to[u + 2 * step] = a2, to[u + 3 * step] = a3;
  }
  for (; u < n16; u += step) to[u] = __ldg(from + u);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned nblocks = gridDim.x * gridDim.y;
    const unsigned done = atomicAdd(p.counter, 1u);
    if (done == nblocks - 1) {  // every block's stores precede this point: publish, then wait
      *p.counter = 0;
      const int dbg = g_push_dbg;
      const int e = *p.epoch;
      if (dbg & 1) {
        __threadfence();
        if (p.lo_dst) *(volatile int*)p.lo_flag = e;
        if (p.hi_dst) *(volatile int*)p.hi_flag = e;
      } else {
        // ONE system-scope release fence (MEMBAR.ALL.SYS, ~2.5 us on B200: the cost of making
        // NVLink stores visible to another GPU), cumulative over every block's stores observed
        // through the counter, then relaxed system-scope flag stores
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        if (p.lo_dst) st_relaxed_sys(p.lo_flag, e);
        if (p.hi_dst) st_relaxed_sys(p.hi_flag, e);
      }
      if (dbg & 2) return;
      // bounded wait (~10 s): a neighbour that never signals sets the error word epoch[1]
      // instead of hanging the device (and later waits fail fast)
      const long long t0 = clock64();
      while (!p.epoch[1] && (p.wait_lo && ld_acquire_sys(p.own) < e) || (p.wait_hi && ld_acquire_sys(p.own + 1) < e)) {
        __nanosleep(128);
        if (clock64() - t0 > 20000000000LL) {
          atomicExch(const_cast<int*>(p.epoch) + 1, e);
          break;
        }
      }
    }
  }
}

__global__ void k_epoch_bump(int* epoch) { *epoch += 1; }
}  // namespace vm

// Depth-phase halo through peer memory (see above).  lo_peer / hi_peer: the neighbours' slab
// bases (same geometry and batch stride as `slab`), null at a global boundary; flags: the
// exchange slot's flag words, own[2] (written by the neighbours), lo_flag = the lo
// neighbour's own[1] word, hi_flag = the hi neighbour's own[0] word; counter: one zeroed
// device word per slot; epoch: the device step counter (vm_halo_epoch_bump).
extern "C" int vm_halo_depth_push(int dtype, const void* slab, int64_t bstride, int B, int C, int D, int H, int W,
                                  void* lo_peer, void* hi_peer, int* lo_flag, int* hi_flag, int* own,
                                  unsigned* counter, const int* epoch, void* stream) {
  VM_REQUIRE(slab && own && counter && epoch, VM_E_ARG, "vm_halo_depth_push: null pointer");
  VM_REQUIRE((!lo_peer || lo_flag) && (!hi_peer || hi_flag), VM_E_ARG, "vm_halo_depth_push: peer without flag");
  VM_REQUIRE(dtype == VM_BF16 || dtype == VM_F32, VM_E_UNSUPPORTED, "vm_halo_depth_push: dtype %d", dtype);
  VM_REQUIRE(D >= 1 && H >= 1 && W >= 1, VM_E_HALO, "vm_halo_depth_push: margin 1 exceeds local extent (%d,%d,%d)",
             D, H, W);
  VM_REQUIRE(((reinterpret_cast<uintptr_t>(slab) | reinterpret_cast<uintptr_t>(lo_peer) |
               reinterpret_cast<uintptr_t>(hi_peer)) & 15) == 0,
             VM_E_ALIGN, "vm_halo_depth_push: 16-byte alignment required");
  const FaceSet s = face_set(dtype, bstride, B, C, D, H, W);
  DepthPush p{};
  p.src = static_cast<const uint8_t*>(slab);
  p.lo_dst = static_cast<uint8_t*>(lo_peer);
  p.hi_dst = static_cast<uint8_t*>(hi_peer);
  p.lo_flag = lo_flag, p.hi_flag = hi_flag, p.own = own, p.counter = counter, p.epoch = epoch;
  p.bstride_b = s.bstride_b, p.plane_b = s.plane_b, p.layer_b = s.plane_b / (D + 2);
  p.B = B, p.CG = s.CG, p.D = D;
  // a neighbour pushes into our margin exactly when we push into its: wait on the same sides
  p.wait_lo = lo_peer != nullptr, p.wait_hi = hi_peer != nullptr;
  const int sides = p.wait_lo + p.wait_hi;
  if (!sides) return VM_OK;
  const int64_t n16 = p.layer_b / 16;
  const int ny = B * s.CG * sides;
  VM_REQUIRE(ny <= 65535 && n16 < (1LL << 31), VM_E_UNSUPPORTED, "vm_halo_depth_push: slab too large");
  int nsm = vm_num_sms(0);
  if (nsm <= 0) nsm = 148;
  // ~4 units per thread, about two waves of 256-thread blocks over the whole exchange
  int64_t gx = (n16 + 256 * 4 - 1) / (256 * 4);
  const int64_t cap = (2 * nsm + ny - 1) / ny;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  launch_pdl(k_depth_push, dim3((unsigned)gx, (unsigned)ny), 256, 0, as_stream(stream), p);
  return launch_status("vm_halo_depth_push");
}

extern "C" void vm_debug_push_mode(int m) { cudaMemcpyToSymbol(g_push_dbg, &m, sizeof(int)); }

extern "C" int vm_halo_epoch_bump(int* epoch, void* stream) {
  VM_REQUIRE(epoch, VM_E_ARG, "vm_halo_epoch_bump: null pointer");
  k_epoch_bump<<<1, 1, 0, as_stream(stream)>>>(epoch);
  return launch_status("vm_halo_epoch_bump");
}

// CUDA-IPC plumbing for the peer mappings: the handle (64 bytes) of the allocation holding
// `ptr` and ptr's offset in it; opening a handle maps the peer allocation once per process
// (cached: a second open of the same allocation returns the first mapping).
extern "C" int vm_ipc_handle(const void* ptr, void* handle64, int64_t* offset) {
  VM_REQUIRE(ptr && handle64 && offset, VM_E_ARG, "vm_ipc_handle: null pointer");
  // the driver entry point through the runtime (libcuda is not a link dependency: the library
  // must load on a host without a driver for the ABI checks)
  typedef CUresult (*range_fn_t)(CUdeviceptr*, size_t*, CUdeviceptr);
  static range_fn_t range_fn = nullptr;
  if (!range_fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range_fn = reinterpret_cast<range_fn_t>(f);
  }
  VM_REQUIRE(range_fn, VM_E_UNSUPPORTED, "vm_ipc_handle: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  VM_REQUIRE(range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) == CUDA_SUCCESS,
             VM_E_ARG, "vm_ipc_handle: not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) cudaGetLastError();
  VM_REQUIRE(e == cudaSuccess, 100 + (int)e, "vm_ipc_handle: cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - (uintptr_t)base);
  return VM_OK;
}

namespace {
struct IpcMap {
  unsigned char key[64];
  void* base;
};
IpcMap g_ipc[512];
int g_nipc = 0;
}  // namespace

extern "C" int vm_ipc_open(const void* handle64, void** base) {
  VM_REQUIRE(handle64 && base, VM_E_ARG, "vm_ipc_open: null pointer");
  for (int i = 0; i < g_nipc; ++i)
    if (!memcmp(g_ipc[i].key, handle64, 64)) {
      *base = g_ipc[i].base;
      return VM_OK;
    }
  VM_REQUIRE(g_nipc < 512, VM_E_UNSUPPORTED, "vm_ipc_open: too many peer allocations");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) cudaGetLastError();  // not sticky: clear it for later launches
  VM_REQUIRE(e == cudaSuccess, 100 + (int)e, "vm_ipc_open: cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  memcpy(g_ipc[g_nipc].key, handle64, 64);
  g_ipc[g_nipc++].base = p;
  *base = p;
  return VM_OK;
}
