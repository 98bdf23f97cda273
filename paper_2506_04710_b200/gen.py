"""Seeded synthetic inputs (include/tbt_gen.h) as numpy arrays.

Complex arrays are numpy complex128 (binary layout of interleaved doubles).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import SIGNATURES, dp, llp
from ._lib import lib as _product_lib

_source = None


def bind(library) -> None:
    """Draws every input from `library` instead of libtbt.so: any shared
    object exporting the tbt_gen.h symbols (oracle/liboracle.so compiles the
    same csrc/gen.cpp, so the values are identical). The reference arm of
    bench.py uses it to keep libtbt.so out of its process."""
    global _source
    if library is not None:
        for name, (res, args) in SIGNATURES.items():
            if name.startswith("tbtgen_"):
                fn = getattr(library, name)
                fn.restype = res
                fn.argtypes = args
    _source = library


def lib():
    return _source if _source is not None else _product_lib()


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous or a.flags.f_contiguous
    return a.ctypes.data_as(dp)


def num_blocks(nx: int, ny: int) -> int:
    return int(lib().tbtgen_num_blocks(nx, ny))


def block_shift(nx: int, ny: int, t: int) -> tuple[int, int]:
    i, j = C.c_int(), C.c_int()
    if lib().tbtgen_block_shift(nx, ny, t, C.byref(i), C.byref(j)):
        raise IndexError(t)
    return i.value, j.value


def blocks(nx: int, ny: int, m: int, seed: int, nthreads: int = 0) -> np.ndarray:
    """Canonical generator blocks, shape (nb, m, m) with [t, a, b] = Z_t(a, b)
    (memory is column-major per block, as the C ABI expects: use
    `blocks_raw` to pass it on)."""
    raw = blocks_raw(nx, ny, m, seed, nthreads)
    return np.transpose(raw, (0, 2, 1))


def blocks_raw(nx: int, ny: int, m: int, seed: int, nthreads: int = 0) -> np.ndarray:
    nb = num_blocks(nx, ny)
    out = np.empty((nb, m, m), dtype=np.complex128)  # [t][b][a] = column-major blocks
    if lib().tbtgen_blocks(nx, ny, m, seed, _ptr(out), nthreads):
        raise ValueError("tbtgen_blocks failed")
    return out


def block_lines(nx: int, ny: int, m: int, seed: int, a: int, nthreads: int = 0):
    """(rows, cols), each (nb, m): rows[t, b] = Z_t(a, b), cols[t, b] = Z_t(b, a)."""
    nb = num_blocks(nx, ny)
    rows = np.empty((nb, m), dtype=np.complex128)
    cols = np.empty((nb, m), dtype=np.complex128)
    if lib().tbtgen_block_lines(nx, ny, m, seed, a, _ptr(rows), _ptr(cols), nthreads):
        raise ValueError("tbtgen_block_lines failed")
    return rows, cols


def correction(m: int, rank: int, seed: int, scale: float = 0.1):
    """(d[40, m], U[40, rank, m], V[40, rank, m]) in the C ABI layout."""
    d = np.empty((40, m), dtype=np.complex128)
    u = np.empty((40, max(rank, 1), m), dtype=np.complex128)
    v = np.empty_like(u)
    if lib().tbtgen_correction(m, rank, seed, scale, _ptr(d), _ptr(u), _ptr(v)):
        raise ValueError("tbtgen_correction failed")
    return d, u[:, :rank].copy(), v[:, :rank].copy()


def rhs_normal(n: int, ncols: int, seed: int) -> np.ndarray:
    out = np.empty((ncols, n), dtype=np.complex128)
    if lib().tbtgen_rhs_normal(n, ncols, seed, _ptr(out)):
        raise ValueError("tbtgen_rhs_normal failed")
    return out.T  # n x ncols, column-major memory


def rhs_delta_steered(nx: int, ny: int, m: int, seed: int, steer_deg: float = 30.0) -> np.ndarray:
    out = np.empty(nx * ny * m, dtype=np.complex128)
    if lib().tbtgen_rhs_delta_steered(nx, ny, m, seed, steer_deg, _ptr(out)):
        raise ValueError("tbtgen_rhs_delta_steered failed")
    return out


def rhs_ports(nx: int, ny: int, m: int, seed: int):
    ne = nx * ny
    out = np.empty((ne, ne * m), dtype=np.complex128)
    rows = np.empty(ne, dtype=np.int64)
    if lib().tbtgen_rhs_ports(nx, ny, m, seed, _ptr(out), rows.ctypes.data_as(llp)):
        raise ValueError("tbtgen_rhs_ports failed")
    return out.T, rows


def component(nx: int, ny: int, r: int, c: int) -> int:
    return int(lib().tbtgen_component(nx, ny, r, c))


def margin(nx: int, ny: int, e, seed: int, scale: float = 0.1):
    """Synthetic margin coupling (tbt_gen.h tbtgen_margin): a Margin with the
    reference-shaped generators bSideGen / bRowGen / bCorner and dense C."""
    from .toeplitz import Margin
    ea = np.ascontiguousarray(e, dtype=np.int32)
    assert ea.size == 9
    ip = C.POINTER(C.c_int)
    ns, nr, nc = C.c_longlong(), C.c_longlong(), C.c_longlong()
    nM = int(lib().tbtgen_margin_lengths(nx, ny, ea.ctypes.data_as(ip), C.byref(ns), C.byref(nr), C.byref(nc)))
    if nM < 0:
        raise ValueError("bad margin sizes")
    bside = np.empty(max(ns.value, 1), np.complex128)
    brow = np.empty(max(nr.value, 1), np.complex128)
    bcorner = np.empty(max(nc.value, 1), np.complex128)
    c = np.empty(max(nM * nM, 1), np.complex128)
    if lib().tbtgen_margin(nx, ny, ea.ctypes.data_as(ip), seed, scale, _ptr(bside), _ptr(brow), _ptr(bcorner),
                           _ptr(c)):
        raise ValueError("tbtgen_margin failed")
    return Margin([int(v) for v in ea], bside[:ns.value], brow[:nr.value], bcorner[:nc.value], c[:nM * nM])
