"""ctypes binding of libtbt.so (include/tbt.h, include/tbt_gen.h).

The library is the product: there is no Python or CPU fallback. Loading
fails loudly when the in-tree build is missing.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtbt.so"

TBT_OK, TBT_USER_ERROR, TBT_NUMERIC_ERROR, TBT_CUDA_ERROR = 0, 1, 2, 3
TBT_HOST, TBT_DEVICE = 0, 1

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
llp = C.POINTER(C.c_longlong)


class TbtDesc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("m", C.c_int), ("max_nrhs", C.c_int),
                ("device", C.c_int), ("flags", C.c_int)]


class TbtGmresOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int),
                ("precondition", C.c_int), ("use_a_only", C.c_int), ("hist_cap", C.c_int),
                ("orthog", C.c_int)]


class TbtGmresStats(C.Structure):
    _fields_ = [("iterations", ip), ("residual", dp), ("converged", ip), ("history", dp),
                ("history_len", ip), ("matvecs", C.c_int)]


class TbtInfo(C.Structure):
    _fields_ = [("n", C.c_longlong), ("bins", C.c_longlong), ("pairs", C.c_longlong),
                ("L0", C.c_int), ("L1", C.c_int), ("spectra_bytes", C.c_longlong),
                ("binprod_kernel", C.c_int), ("kernels_per_apply", C.c_int),
                ("has_antisym", C.c_int), ("apply_path", C.c_int)]


# name -> (restype, argtypes); the exported C ABI of tbt.h and tbt_gen.h.
SIGNATURES = {
    "tbt_create": (C.c_int, [C.POINTER(TbtDesc), C.POINTER(C.c_void_p)]),
    "tbt_destroy": (None, [C.c_void_p]),
    "tbt_last_error": (C.c_char_p, []),
    "tbt_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tbt_get_stream": (C.c_void_p, [C.c_void_p]),
    "tbt_set_generators": (C.c_int, [C.c_void_p, dp, C.c_longlong]),
    "tbt_set_generators_full": (C.c_int, [C.c_void_p, dp, C.c_longlong]),
    "tbt_set_correction": (C.c_int, [C.c_void_p, C.c_int, dp, dp, dp]),
    "tbt_precompute": (C.c_int, [C.c_void_p]),
    "tbt_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "tbt_apply_many": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong]),
    "tbt_apply_a": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "tbt_apply_b": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "tbt_apply_bt": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "tbt_apply_c": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "tbt_diagonal": (C.c_int, [C.c_void_p, dp]),
    "tbt_size_a": (C.c_longlong, [C.c_void_p]),
    "tbt_size_m": (C.c_longlong, [C.c_void_p]),
    "tbt_set_margin": (C.c_int, [C.c_void_p, ip, dp, dp, dp, dp]),
    "tbt_set_margin_dense": (C.c_int, [C.c_void_p, ip, dp, dp]),
    "tbt_ztoe1_mode": (C.c_int, [C.c_char_p, ip]),
    "tbt_ztoe1_read_dense": (C.c_int, [C.c_char_p, dp, dp, dp]),
    "tbt_gmres": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(TbtGmresOpts),
                            C.POINTER(TbtGmresStats), C.c_int]),
    "tbt_schur_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(TbtGmresOpts),
                                  C.POINTER(TbtGmresStats), C.c_int]),
    "tbt_load_ztoe1": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "tbt_ztoe1_dims": (C.c_int, [C.c_char_p, ip, ip, ip]),
    "tbt_ztoe1_read": (C.c_int, [C.c_char_p, dp, dp, dp, dp, dp]),
    "tbt_set_cache_key": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    "tbt_save_spectra": (C.c_int, [C.c_void_p, C.c_char_p]),
    "tbt_load_spectra": (C.c_int, [C.c_void_p, C.c_char_p]),
    "tbt_port_network": (C.c_int, [C.c_void_p, dp, C.c_longlong, C.c_int, llp, C.c_double, dp, dp, dp, dp, C.c_int]),
    "tbt_array_farfield": (C.c_int, [C.c_void_p, C.POINTER(dp), C.POINTER(dp), ip, C.c_int, dp, C.c_double,
                                     C.c_double, C.c_double, C.c_double, dp, C.c_int, dp, C.c_int, dp, dp, C.c_int]),
    "tbt_get_info": (C.c_int, [C.c_void_p, C.POINTER(TbtInfo)]),
    "tbt_get_spectrum_bin": (C.c_int, [C.c_void_p, C.c_longlong, dp]),
    "tbt_bench_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, dp, dp]),
    "tbt_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "tbt_dist_unique_id": (C.c_int, [C.c_char_p]),
    "tbt_dist_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_char_p]),
    "tbt_dist_init_loopback": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_char_p]),
    "tbt_dist_transport": (C.c_int, [C.c_void_p, ip]),
    "tbt_dist_rows": (C.c_int, [C.c_void_p, ip, ip]),
    "tbt_dist_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, ip, ip, ip, ip]),
    "tbt_phase_times": (C.c_int, [C.c_void_p, C.c_int, dp]),
    "tbt_cta_trace": (C.c_int, [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_longlong, llp]),
    "tbt_timing_read": (C.c_int, [C.c_void_p, dp, ip]),
    "tbtgen_num_blocks": (C.c_longlong, [C.c_int, C.c_int]),
    "tbtgen_block_shift": (C.c_int, [C.c_int, C.c_int, C.c_longlong, ip, ip]),
    "tbtgen_blocks": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, dp, C.c_int]),
    "tbtgen_block_lines": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, dp, dp, C.c_int]),
    "tbtgen_correction": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_double, dp, dp, dp]),
    "tbtgen_rhs_normal": (C.c_int, [C.c_longlong, C.c_int, C.c_uint64, dp]),
    "tbtgen_rhs_delta_steered": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, dp]),
    "tbtgen_rhs_ports": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, dp, llp]),
    "tbtgen_component": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "tbtgen_margin_size": (C.c_longlong, [C.c_int, C.c_int, ip]),
    "tbtgen_margin_lengths": (C.c_longlong, [C.c_int, C.c_int, ip, llp, llp, llp]),
    "tbtgen_margin": (C.c_int, [C.c_int, C.c_int, ip, C.c_uint64, C.c_double, dp, dp, dp, dp]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().tbt_last_error()
    return msg.decode() if msg else ""
