"""ctypes binding of libttsvd_cu.so — the C-ABI declared in include/ttsvd_cu.h.

The library is the product: if it is missing this module raises instead of
falling back to anything else.  Build it with ``python -m
paper_2102_00104_b200.build`` (``__graft_entry__.build()`` does it too).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("TTSVD_LIB_VARIANT") or os.path.join(HERE, "libttsvd_cu.so")  # override: diagnostics builds
HEADER = os.path.join(ROOT, "include", "ttsvd_cu.h")

i64 = C.c_int64
dptr = C.c_void_p  # device or host pointer as an integer address
i64p = C.POINTER(C.c_int64)


class Step(C.Structure):
    _fields_ = [("rows", i64), ("cols", i64), ("nsig", i64), ("rank", i64),
                ("t_tsqr_ms", C.c_double), ("t_svd_ms", C.c_double), ("t_tsmm_ms", C.c_double),
                ("t_tsqr_sweep_ms", C.c_double), ("tsqr_kernel", C.c_int32), ("svd_sweeps", C.c_int32),
                ("t_reorder_ms", C.c_double)]


TSQR_KERNELS = {0: "none", 1: "tsqr_ws_kernel", 2: "tsqr_tile_kernel", 3: "tsqr_la_kernel", 4: "tsqr_t128_kernel",
                5: "gqr_kernel", 6: "tsqr_pt_kernel",
                7: "tsqr_gs_kernel", 8: "tsqr_t128_kernel (tile levels)", 9: "tsqr_gt_kernel"}


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, i64, C.c_void_p)

_SIGS = {
    "ttsvd_cu_version": (C.c_char_p, []),
    "ttsvd_cu_last_error": (C.c_char_p, []),
    "ttsvd_cu_ctx_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ttsvd_cu_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ttsvd_cu_synchronize": (C.c_int, [C.c_void_p]),
    "ttsvd_cu_ctx_launches": (i64, [C.c_void_p]),
    "ttsvd_cu_ctx_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "ttsvd_cu_padded_stride": (i64, [i64]),
    "ttsvd_cu_tsqr": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, dptr]),
    "ttsvd_cu_reduce_block": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, dptr, i64, dptr]),
    "ttsvd_cu_combine_factors": (C.c_int, [C.c_void_p, dptr, i64, i64, dptr]),
    "ttsvd_cu_small_svd": (C.c_int, [C.c_void_p, dptr, i64, dptr, dptr]),
    "ttsvd_cu_jacobi_svd": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, dptr, dptr, dptr]),
    "ttsvd_cu_driver_svd": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, i64, dptr, dptr, C.POINTER(C.c_int32)]),
    "ttsvd_cu_select_rank": (C.c_int, [C.c_void_p, dptr, i64, C.c_double, i64, i64p]),
    "ttsvd_cu_select_rank_host": (i64, [C.c_void_p, i64, C.c_double, i64]),
    "ttsvd_cu_derive_delta": (C.c_int, [C.c_double, C.c_double, i64, C.POINTER(C.c_double)]),
    "ttsvd_cu_tsmm_reshape": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, dptr, i64, i64, dptr, i64, i64, i64]),
    "ttsvd_cu_tt_svd": (C.c_int, [C.c_void_p, dptr, i64p, i64, i64, i64, C.c_double, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_run_chain": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, i64p, i64, i64, C.c_double, i64,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_void_p)]),
    "ttsvd_cu_tt_svd_two_sided": (C.c_int, [C.c_void_p, dptr, i64p, i64, i64, i64, C.c_double,
                                            C.POINTER(C.c_void_p)]),
    "ttsvd_cu_transpose_reorder": (C.c_int, [C.c_void_p, dptr, i64, i64, i64, dptr, i64, i64, i64]),
    "ttsvd_cu_choose_combined_dims": (C.c_int, [i64p, i64, i64, C.c_double, C.c_void_p, i64, i64, i64p, i64p]),
    "ttsvd_cu_tt_svd_thick": (C.c_int, [C.c_void_p, C.c_void_p, i64p, i64, i64, i64, C.c_double, i64, C.c_double,
                                        C.c_void_p, i64, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_tt_svd_thick_host": (C.c_int, [C.c_void_p, C.c_void_p, i64p, i64, i64, i64, C.c_double, i64, C.c_double,
                                             C.c_void_p, i64, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_tt_svd_host": (C.c_int, [C.c_void_p, dptr, i64p, i64, i64, i64, C.c_double, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_tt_svd_distributed": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), i64, i64, i64, i64p, i64, i64, i64,
                                              C.c_double, EXCHANGE_FN, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_comm_unique_id": (C.c_int, [C.c_void_p]),
    "ttsvd_cu_ctx_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "ttsvd_cu_ctx_comm_init_all": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "ttsvd_cu_tt_svd_distributed_devices": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p), i64, i64p,
                                                      i64, i64, i64, C.c_double, C.POINTER(C.c_void_p)]),
    "ttsvd_cu_gen_partition": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.c_double, i64, i64, i64, i64, i64, dptr]),
    "ttsvd_cu_tt_d": (i64, [C.c_void_p]),
    "ttsvd_cu_tt_ranks": (C.c_int, [C.c_void_p, i64p]),
    "ttsvd_cu_tt_core": (C.c_int, [C.c_void_p, i64, C.c_void_p]),
    "ttsvd_cu_tt_nsteps": (i64, [C.c_void_p]),
    "ttsvd_cu_tt_step": (C.c_int, [C.c_void_p, i64, C.POINTER(Step)]),
    "ttsvd_cu_tt_sigma": (C.c_int, [C.c_void_p, i64, C.c_void_p]),
    "ttsvd_cu_tt_free": (None, [C.c_void_p]),
    "ttsvd_cu_gen_uniform": (C.c_int, [C.c_void_p, C.c_uint64, i64, i64, i64, dptr]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)  # drop comments
    return sorted(set(re.findall(r"\b(ttsvd_cu_[a-z_0-9]+)\s*\(", txt)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build the CUDA library with "
                               "`python -m paper_2102_00104_b200.build` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
