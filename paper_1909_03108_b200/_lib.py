"""ctypes binding of libvoxmesh_sm100.so (the C ABI declared in include/vm_api.h).

The product path has no CPU fallback: if the library is missing, or CUDA is not
available when a kernel is called, the call raises.  Every wrapper passes raw
device pointers (``tensor.data_ptr()``), explicit sizes and the current torch
CUDA stream, and maps negative return codes to the reference's exception types.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import HaloError, ShardingError, VoxmeshError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvoxmesh_sm100.so")

VM_F32, VM_BF16, VM_F64, VM_U8 = 0, 1, 2, 3
VM_CONV_RELU, VM_CONV_MASK, VM_CONV_NOBIAS = 1, 2, 4

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_F = ctypes.c_float
_U = ctypes.c_uint
_S = ctypes.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "vm_version": (_I, []),
    "vm_error_string": (ctypes.c_char_p, [_I]),
    "vm_last_error": (ctypes.c_char_p, []),
    "vm_num_sms": (_I, [_I]),
    "vm_launch_count": (ctypes.c_longlong, []),
    "vm_set_pdl": (ctypes.c_int, [ctypes.c_int]),
    "vm_set_conv_sm_limit": (ctypes.c_int, [ctypes.c_int]),
    "vm_box_pack": (_I, [_P, _c_i64p, _I, _c_i64p, _c_i64p, _P, _P]),
    "vm_box_unpack": (_I, [_P, _c_i64p, _I, _c_i64p, _c_i64p, _P, _P]),
    "vm_box_unpack_add": (_I, [_P, _c_i64p, _I, _c_i64p, _c_i64p, _P, _P]),
    "vm_box_zero": (_I, [_P, _c_i64p, _I, _c_i64p, _c_i64p, _P]),
    "vm_dense_to_slab": (_I, [_P, _I, _P, _I, _L, _I, _I, _I, _I, _I, _I, _P]),
    "vm_slab_to_dense": (_I, [_P, _I, _L, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "vm_onehot_u8": (_I, [_P, _P, _L, _I, _P]),
    "vm_conv3d_fwd_simt": (_I, [_I, _P, _L, _P, _P, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _U, _P]),
    "vm_conv3d_wgrad_simt_ws": (ctypes.c_size_t, [_I, _I, _I, _I, _I, _I]),
    "vm_conv3d_wgrad_simt": (_I, [_I, _P, _L, _P, _L, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "vm_weight_flip_transpose": (_I, [_P, _P, _I, _I, _I, _P]),
    "vm_packed_weights_bytes": (ctypes.c_size_t, [_I, _I]),
    "vm_pack_weights": (_I, [_P, _P, _I, _I, _I, _P]),
    "vm_pack_weights_batch": (_I, [_P, _I, _L, _P]),
    "vm_conv3d_fwd_tc": (_I, [_P, _L, _P, _P, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _U, _P]),
    "vm_conv3d_fwd_tc_ws": (_I, [_P, _L, _P, _P, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _U, _P, _S, _P]),
    "vm_conv3d_fwd_tc_ws_bytes": (_S, [_I, _I, _I, _I, _I, _I]),
    "vm_conv3d_fwd_c1": (_I, [_P, _L, _P, _P, _P, _L, _I, _I, _I, _I, _I, _U, _P]),
    "vm_conv3d_wgrad_c1_ws": (_S, [_I, _I, _I, _I, _I]),
    "vm_dense_to_compact1": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "vm_aug_stats_ws_bytes": (_S, []),
    "vm_aug_stats": (_I, [_P, _P, _L, _P, _P, _P]),
    "vm_aug_remove": (_I, [_P, _P, _L, _F, _P]),
    "vm_aug_count_chunks": (_I, [_P, _L, _I, _I, _P, _P]),
    "vm_aug_paint": (_I, [_P, _I, _I, _I, _P, _P, _I, _P, _P]),
    "vm_aug_blur_axis": (_I, [_P, _P, _I, _I, _I, _I, _P, _I, _P]),
    "vm_aug_finish": (_I, [_P, _P, _P, _L, _F, _F, _P]),
    "vm_conv3d_wgrad_c1": (_I, [_P, _L, _P, _L, _P, _P, _P, _I, _I, _I, _I, _I, _P]),
    "vm_conv3d_wgrad_tc_ws": (ctypes.c_size_t, [_I, _I, _I, _I, _I, _I]),
    "vm_conv3d_wgrad_tc": (_I, [_P, _L, _P, _L, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "vm_conv3d_wgrad_tc_deferrable": (_I, [_I, _I, _I, _I, _I, _I]),
    "vm_conv3d_wgrad_tc_phase": (_I, [_P, _L, _P, _L, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "vm_maxpool2_fwd": (_I, [_I, _P, _L, _P, _L, _I, _I, _I, _I, _I, _P]),
    "vm_maxpool2_bwd": (_I, [_I, _P, _L, _P, _L, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _P]),
    "vm_upsample2_fwd": (_I, [_I, _P, _L, _P, _L, _I, _I, _I, _I, _I, _P]),
    "vm_upsample2_bwd": (_I, [_I, _P, _L, _P, _L, _P, _L, _I, _I, _I, _I, _I, _P]),
    "vm_relu_mask": (_I, [_I, _P, _L, _P, _L, _P, _L, _I, _I, _I, _I, _I, _P]),
    "vm_head_partials_count": (_I, [_I, _I, _I, _I]),
    "vm_head_fwd": (_I, [_I, _P, _L, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _F, _P]),
    "vm_reduce_rows": (_I, [_P, _I, _I, _P, _P]),
    "vm_label_counts": (_I, [_P, _P, _L, _I, _P, _P]),
    "vm_head_bwd": (_I, [_I, _P, _L, _P, _P, _P, _P, _P, _L, _P, _I, _I, _I, _I, _I, _I, _F, _F, _F, _I, _F, _I, _P]),
    "vm_head_bwd_dprobs": (_I, [_I, _P, _L, _P, _P, _P, _P, _L, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "vm_softmax_rows": (_I, [_I, _P, _P, _L, _I, _P]),
    "vm_concat_rows": (_I, [_P, _L, _P, _L, _P, _L, _P]),
    "vm_loss_stats": (_I, [_P, _P, _L, _I, _F, _P, _P, _P]),
    "vm_loss_grad": (_I, [_P, _P, _P, _L, _I, _F, _F, ctypes.c_double, _I, _F, _P, _P]),
    "vm_sgd_momentum": (_I, [_P, _P, _P, _P, _I, _L, _P, _F, _F, _P]),
    "vm_nccl_bind": (_I, []),
    "vm_halo_slab_ws_bytes": (_S, [_I, _I, _I, _I, _I, _I]),
    "vm_halo_slab_fwd": (_I, [_P, _I, _P, _L, _I, _I, _I, _I, _I, _P, _P, _S, _P, _P]),
    "vm_set_halo_zero_copy_min": (ctypes.c_longlong, [ctypes.c_longlong]),
    "vm_halo_slab_zero": (_I, [_I, _P, _L, _I, _I, _I, _I, _I, _P, _P]),
    "vm_halo_slab_pack": (_I, [_I, _P, _L, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "vm_halo_slab_unpack": (_I, [_I, _P, _L, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "vm_halo_slab_face_bytes": (ctypes.c_longlong, [_I, _I, _I, _I, _I, _I, _I]),
    "vm_allreduce_f32": (_I, [_P, _P, _S, _P]),
    "vm_halo_depth_push": (_I, [_I, _P, _L, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vm_halo_epoch_bump": (_I, [_P, _P]),
    "vm_ipc_handle": (_I, [_P, _P, _P]),
    "vm_ipc_open": (_I, [_P, _P]),
    "vm_conv3d_fwd_tc_link": (_I, [_P, _L, _P, _P, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _U, _P, _S, _P, _P]),
    "vm_conv3d_fwd_tc_range": (_I, [_P, _L, _P, _P, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _I, _I, _U, _P, _S,
                                    _P]),
    # SURVEY §8(b) composites (csrc/abi.cu)
    "vm_conv3d_dgrad": (_I, [_P, _L, _P, _P, _L, _P, _L, _I, _I, _I, _I, _I, _I, _P]),
}

# entry points declared in include/vm_api.h (the ABI test checks each is exported)
EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


class LibraryMissing(VoxmeshError):
    """libvoxmesh_sm100.so was not built or cannot be loaded."""


def load():
    """Load (once) and return the shared library; raise LibraryMissing otherwise."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def missing_symbols():
    lib = load()
    return [n for n in EXPORTED if getattr(lib, n, None) is None]


def _raise(code, name):
    lib = load()
    detail = (lib.vm_last_error() or b"").decode(errors="replace")
    text = f"{name}: {lib.vm_error_string(code).decode()} ({detail})"
    if code == -5:
        raise HaloError(detail or text)
    if code == -3 and "even local extents" in detail:
        from .errors import GraphBuildError

        raise GraphBuildError(detail)
    if code < 0:
        raise VoxmeshError(text)
    raise VoxmeshError(f"CUDA failure in {text}")


def call(name, *args):
    """Invoke an entry point; raises on a non-zero status."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        _raise(rc, name)
    return rc


def call_size(name, *args):
    """Invoke a size-returning entry point (no status code)."""
    return getattr(load(), name)(*args)


def i64arr(vals):
    arr = (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
    return arr


def stream_ptr(stream=None):
    import torch

    if not torch.cuda.is_available():
        raise VoxmeshError("CUDA device required: the B200 path has no CPU fallback")
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def dtype_code(torch_dtype):
    import torch

    table = {torch.float32: VM_F32, torch.bfloat16: VM_BF16, torch.float64: VM_F64, torch.uint8: VM_U8}
    if torch_dtype not in table:
        raise ShardingError(f"unsupported dtype {torch_dtype}")
    return table[torch_dtype]
