// abi.cu — the entry-point names of the SURVEY §8(b) ABI sketch, as thin wrappers over the
// kernels' own entry points (same stream-ordered, non-allocating, return-code contract).
// The halo transport and the all-reduce stay in torch.distributed / NCCL on the Python side
// (paper_1909_03108_b200/mesh.py), so vm_init / vm_comm_split / vm_allreduce_f32 and the
// NCCL half of vm_halo_fwd/bwd have no C counterpart; the device half (face pack / unpack /
// unpack-add of a padded block) is vm_box_pack / vm_box_unpack / vm_box_unpack_add (box.cu).
#include "vm_common.cuh"

using namespace vm;

// conv3d_local (ops.py:69-97): y = [relu](conv(x) + bias), packed forward operand
extern "C" int vm_conv3d_fwd(const void* x, int64_t x_bstride, const void* wpacked, const float* bias,
                             void* y, int64_t y_bstride, int B, int Cin, int Cout, int D, int H, int W,
                             unsigned flags, void* stream) {
  VM_REQUIRE(!(flags & VM_CONV_MASK), VM_E_ARG, "vm_conv3d_fwd: use vm_conv3d_dgrad for masked output");
  return vm_conv3d_fwd_tc(x, x_bstride, wpacked, bias, y, y_bstride, nullptr, 0, B, Cin, Cout, D, H, W,
                          flags, stream);
}

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

// conv3d_param_grads_local (ops.py:117-138)
extern "C" size_t vm_conv3d_wgrad_ws(int B, int Cin, int Cout, int D, int H, int W) {
  return vm_conv3d_wgrad_tc_ws(B, Cin, Cout, D, H, W);
}
extern "C" int vm_conv3d_wgrad(const void* x, int64_t x_bstride, const void* gy, int64_t gy_bstride, float* gw,
                               float* gb, void* ws, int B, int Cin, int Cout, int D, int H, int W, void* stream) {
  return vm_conv3d_wgrad_tc(x, x_bstride, gy, gy_bstride, gw, gb, ws, B, Cin, Cout, D, H, W, stream);
}

// relu_backward_local (ops.py:186-187)
extern "C" int vm_relu_bwd(int dtype, const void* g, int64_t g_bstride, const void* mask, int64_t mask_bstride,
                           void* out, int64_t out_bstride, int B, int C, int D, int H, int W, void* stream) {
  return vm_relu_mask(dtype, g, g_bstride, mask, mask_bstride, out, out_bstride, B, C, D, H, W, stream);
}

// upsample2 (ops.py:171-173) written straight into the up half of the decoder concat slab
// (unet.py:215): y = the concat slab's first channel group, y_bstride = the concat slab's
// batch stride.
extern "C" int vm_upsample2_concat_fwd(int dtype, const void* x, int64_t x_bstride, void* y_concat,
                                       int64_t y_bstride, int B, int C, int D, int H, int W, void* stream) {
  return vm_upsample2_fwd(dtype, x, x_bstride, y_concat, y_bstride, B, C, D, H, W, stream);
}

// head 1x1x1 conv + softmax + loss statistics (unet.py:223, ops.py:190-194, training.py:77-92)
extern "C" int vm_head_softmax_stats(int dtype, const void* y, int64_t y_bstride, const float* w,
                                     const float* b, const float* onehot, float* probs, float* partials,
                                     int B, int C, int ncls, int D, int H, int W, float clamp, void* stream) {
  return vm_head_fwd(dtype, y, y_bstride, w, b, onehot, probs, partials, B, C, ncls, D, H, W, clamp, stream);
}

// loss gradient (training.py:110-127) -> softmax backward -> head backward
extern "C" int vm_loss_grad_head_bwd(int dtype, const void* y, int64_t y_bstride, const float* w,
                                     const float* b, const float* onehot, const float* stats, void* g,
                                     int64_t g_bstride, float* wpartials, int B, int C, int ncls, int D, int H,
                                     int W, float w_dice, float w_ce, float total_voxels, int dice_mask,
                                     float clamp, int relu_mask, void* stream) {
  return vm_head_bwd(dtype, y, y_bstride, w, b, onehot, stats, g, g_bstride, wpartials, B, C, ncls, D, H, W,
                     w_dice, w_ce, total_voxels, dice_mask, clamp, relu_mask, stream);
}
