"""ctypes binding of libgzccl.so (include/gzccl.h).

There is no fallback: if the CUDA library is missing or no CUDA device is
present, every codec / collective call raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GZCCL_LIB") or os.path.join(HERE, "libgzccl.so")  # override: A/B experiments

GZ_OK = 0
GZ_EINVAL = 10001
GZ_EBOUND = 10002
GZ_ECAPACITY = 10003
GZ_EBLOCK = 10004

# exported symbols (include/gzccl.h) -> (restype, argtypes)
u64, u32, i32, p, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
SIGNATURES = {
    "gz_compress_bound": (u64, [u64]),
    "gz_num_tiles": (u64, [u64]),
    "gz_tile_blocks": (u32, []),
    "gz_sidecar_bytes": (u64, [u64]),
    "gz_workspace_bytes": (u64, [u64]),
    "gz_workspace_init": (i32, [p, u64, p]),
    "gz_status_reset": (i32, [p, p]),
    "gz_compress": (i32, [p, u64, dbl, u32, p, u64, p, p, p, p, u64, p, p]),
    "gz_decompress_sidecar": (i32, [p, p, u64, dbl, p, p, p]),
    "gz_decompress_reduce": (i32, [p, p, p, u64, dbl, i32, p, p, p]),
    "gz_decompress_multi": (i32, [p, p, p, u32, dbl, p, i32, p, p]),
    "gz_decompress_slots_multi": (i32, [p, p, p, p, u32, dbl, p, i32, p, p]),
    "gz_index": (i32, [p, u64, u64, p, p, u64, p, p]),
    "gz_index_workspace_bytes": (u64, [u64]),
    "gz_reduce_step": (i32, [p, p, p, u64, dbl, i32, p, p, u64, p, p, p, u64, p, p]),
    "gz_segments_workspace_bytes": (u64, [p, u32]),
    "gz_compress_segments": (i32, [p, p, u32, dbl, p, p, p, p, p, p, p, u64, p, p]),
    "gz_ipc_handle_size": (i32, []),
    "gz_ipc_get_handle": (i32, [p, p]),
    "gz_ipc_open_handle": (i32, [p, ctypes.POINTER(ctypes.c_void_p)]),
    "gz_ipc_close": (i32, [p]),
    "gz_enable_peer_access": (i32, [i32]),
    "gz_stream_write_u32": (i32, [p, p, u32]),
    "gz_stream_wait_u32_geq": (i32, [p, p, u32]),
    "gz_stream_flag_ops": (i32, [p, p, u32]),
    "gz_copy_blob": (i32, [p, p, p, u64, p]),
    "gz_copy_items": (i32, [p, u32, p]),
    "gz_copy_checked": (i32, [p, p, u64, u64, p, p]),
    "gz_apply_op": (i32, [p, p, p, u64, i32, p]),
    "gz_status_key": (i32, [p, i32, p, p]),
    "gz_copy_items_sms": (i32, [p, u32, i32, p]),
    "gz_launch_count": (u64, []),
    "gz_debug_stamp": (i32, [p, p]),
    "gz_slots_bytes": (u64, [u64]),
    "gz_step": (i32, [p, p, u64, dbl, i32, p, p, u64, p, p]),
    "gz_step_reduce": (i32, [p, p, u64, dbl, i32, p, p, p]),
    "gz_fr_bound": (u64, [u64, u32]),
    "gz_fr_workspace_bytes": (u64, []),
    "gz_fr_compress": (i32, [p, u64, u32, p, u64, p, p, p, p]),
    "gz_fr_decompress": (i32, [p, u64, u32, p, p]),
}

_lib = None


class GzError(RuntimeError):
    pass


def lib():
    """Load libgzccl.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2308_05199_b200.build` "
                               "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == GZ_OK:
        return
    if rc == GZ_EBOUND:
        raise ValueError(f"{what}: error bound must be positive and finite")
    if rc == GZ_EBLOCK:
        raise ValueError(f"{what}: block size must be 32 (frozen format, codec.py:42)")
    if rc in (GZ_EINVAL, GZ_ECAPACITY):
        raise ValueError(f"{what}: invalid argument (code {rc})")
    raise GzError(f"{what}: CUDA error {rc}")
