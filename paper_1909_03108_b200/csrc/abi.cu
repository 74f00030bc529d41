// abi.cu — composite entry points of the SURVEY §8(b) ABI that add logic over the kernels'
// own entry points (same stream-ordered, non-allocating, return-code contract).
#include "vm_common.cuh"

using namespace vm;

// conv3d_input_grad_local (ops.py:100-114) fused with relu_backward_local (ops.py:186-187):
// gx = conv(gy_halo, flip(W)^T) [* (mask > 0)]; wpacked_t = vm_pack_weights(.., flip=1);
// Cin/Cout are the FORWARD conv's (gx has Cin channels).  mask may be NULL.
extern "C" int vm_conv3d_dgrad(const void* gy, int64_t gy_bstride, const void* wpacked_t, const void* mask,
                               int64_t mask_bstride, void* gx, int64_t gx_bstride, int B, int Cin, int Cout,
                               int D, int H, int W, void* stream) {
  const unsigned flags = VM_CONV_NOBIAS | (mask ? VM_CONV_MASK : 0u);
  return vm_conv3d_fwd_tc(gy, gy_bstride, wpacked_t, nullptr, gx, gx_bstride, mask, mask_bstride, B, Cout, Cin,
                          D, H, W, flags, stream);
}

