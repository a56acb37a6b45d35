"""ctypes binding of ``libagile_b200.so`` (the C-ABI in ``include/agile_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is no CPU
fallback: loading fails loudly when the library is missing, and ``agile_create`` fails when no
GPU is visible.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import CODE_TO_EXC, NativeUnavailable

LIB_PATH = os.environ.get("AGILE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libagile_b200.so")

_u32, _u64, _i64, _int, _vp, _cp = C.c_uint32, C.c_uint64, C.c_int64, C.c_int, C.c_void_p, C.c_char_p
_pu32, _pu64, _pi64, _pi8, _pf = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int8), C.POINTER(C.c_float))

# name -> (restype, argtypes); pointer arguments are passed as c_void_p (raw addresses) so callers
# can hand over numpy buffers, torch data_ptr()s and pinned host memory alike.
SIGNATURES = {
    "agile_create": (_int, [_cp, _int, C.POINTER(_vp)]),
    "agile_destroy": (_int, [_vp]),
    "agile_last_error": (_cp, [_vp]),
    "agile_geometry": (_int, [_vp, _vp, _int]),
    "agile_store_attach": (_int, [_vp, _int, _vp, _u64, _cp]),
    "agile_store_ptr": (_int, [_vp, _int, C.POINTER(_vp), C.POINTER(_u64)]),
    "agile_store_fill": (_int, [_vp, _int, _u64, _u64, _u64, _int]),
    "agile_store_load_image": (_int, [_vp, _int, _cp]),
    "agile_store_save_image": (_int, [_vp, _int, _cp]),
    "agile_reset": (_int, [_vp, _int]),
    "agile_stats": (_int, [_vp, _vp, _int]),
    "agile_trace_enable": (_int, [_vp, _u64]),
    "agile_event_log": (_int, [_vp, _vp, _u64, C.POINTER(_u64)]),
    "agile_sync": (_int, [_vp, _vp]),
    "agile_run_seq": (_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "agile_run_reads": (_int, [_vp, _vp, _u32, _u32, _u32, _int, _u64, _vp, _vp, _vp, _vp]),
    "agile_run_loop": (_int, [_vp, _u32, _u64, _u64, _u64, _vp, _vp, _vp]),
    "agile_run_gather": (_int, [_vp, _vp, _u32, _u32, _u32, _int, _u64, _vp, _vp, _vp]),
    "agile_embbag": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u32, _u32, _u32, _u32, _u32, _u32, _u32, _vp]),
    "agile_run_loop_rw": (_int, [_vp, _u32, _u64, _u64, _u64, _vp, _vp, _int, _vp]),
    "agile_write_blocks": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "agile_evict_blocks": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "agile_array_get": (_int, [_vp, _vp, _vp, _i64, _u32, _vp]),
    "agile_set_launch_mode": (_int, [_vp, _int]),
    "agile_set_engine_copy": (_int, [_vp, _int]),
    "agile_user_run_begin": (_int, [_vp, _vp, _u32, _u64, _vp, _u64, _vp, _u64, C.POINTER(_vp)]),
    "agile_user_run_end": (_int, [_vp, _vp]),
    "agile_flush": (_int, [_vp, C.POINTER(_u64)]),
    "agile_lock_cycle_demo": (_int, [_vp, _u32, _int]),
    "agile_buffer_busy_demo": (_int, [_vp, _int]),
    "agile_share_live": (_int, [_vp, C.POINTER(_u64)]),
    "agile_run_coherence": (_int, [_vp, _vp, _vp, _vp, _u32, _u32, _vp, C.POINTER(_u64)]),
    "agile_embbag_host_submit": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u32, _u32, _u32, _u32, _u32, _int]),
    "agile_embbag_host_wait": (_int, [_vp, _int]),
    "agile_embbag_ctas": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u32, _u32, _u32, _u32, _u32, _u32, _u32, _u32, _vp]),
    "agile_embbag_host": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u32, _u32, _u32, _u32, _u32]),
    "agile_embbag_grid": (_int, [_vp, C.POINTER(_u32), C.POINTER(_u32)]),
    "agile_bfs": (_int, [_vp, _vp, _u32, _u32, _u64, _vp, _u32, _vp, _vp]),
    "agile_spmv": (_int, [_vp, _vp, _u32, _u64, _u64, _u64, _vp, _vp, C.c_float, C.c_float, _u32, _vp, _vp]),
    "agile_embbag_prefetch": (_int, [_vp, _vp, _vp, _vp, _vp, _u32, _u32, _u32, _u32, _u32, _vp]),
    "agile_embbag_sharded": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _u32, _u32, _u32, _u32, _u32, _u32, _int,
                                    _vp]),
    "agile_store_fill_rows": (_int, [_vp, _int, _u64, _u64, _u32, _u64, _u64, _u32]),
    "agile_spmv_rows": (_int, [_vp, _vp, _u32, _u64, _u32, _u64, _u64, _vp, _vp, C.c_float, C.c_float, _u32, _vp,
                               _vp]),
    "agile_bfs_level": (_int, [_vp, _vp, _u32, _vp, _u32, _vp, _vp, _vp, C.c_int32, _u64, _u32, _vp, _vp]),
}

_lib = None


def load():
    """Load the native library once; raise NativeUnavailable if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (the B200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(ctx, rc: int, what: str = "") -> None:
    """Map a negative return code to the reference exception type."""
    if rc == 0:
        return
    msg = load().agile_last_error(ctx)
    msg = msg.decode() if msg else ""
    exc = CODE_TO_EXC.get(rc, RuntimeError)
    raise exc(f"{what}: {msg} (rc={rc})" if what else f"{msg} (rc={rc})")
