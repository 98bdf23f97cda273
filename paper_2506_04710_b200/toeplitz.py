"""Host-side mirror of the reference's operator and solver API
(proj/include/arraymom/linsolve.hpp:26-95) over the C ABI of libtbt.so.

    ToeplitzMatvec(rep)      -> ToeplitzMatvec(rep, model)   linsolve.hpp:61
      .apply / .applyA / .diagonal / .sizeA / .sizeM          linsolve.hpp:64-72
    toeplitz_matvec(rep, x)  -> toeplitzMatvec               linsolve.hpp:80-81
    iterative_solve(rep, V, opt) -> iterativeSolve           linsolve.hpp:88-89
    SolverOptions / SolveResult / UserError / NumericError   linsolve.hpp:40-53,
                                                             common.hpp:38-50

`ToeplitzRep` here holds what the hot path consumes from the reference's
ToeplitzRep (toeplitz.hpp:67-107): nx, ny, e5 = m and the Sparse A
generators aGen (toeplitz.hpp:72-74), plus the synthetic nine-component
correction that stands in for the margin blocks of the BASELINE workloads.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import TBT_DEVICE, TBT_HOST, TbtDesc, TbtGmresOpts, TbtGmresStats, TbtInfo, dp, lib


class UserError(RuntimeError):
    """Bad input (reference UserError, exit code 1)."""


class NumericError(RuntimeError):
    """Numerical failure, e.g. GMRES non-convergence (reference NumericError, exit code 2)."""


class DeviceError(RuntimeError):
    """CUDA failure or no usable sm_100 device."""


def _check(status: int) -> None:
    if status == _lib.TBT_OK:
        return
    msg = _lib.last_error()
    if status == _lib.TBT_USER_ERROR:
        raise UserError(msg)
    if status == _lib.TBT_NUMERIC_ERROR:
        raise NumericError(msg)
    raise DeviceError(msg)


@dataclass
class Correction:
    rank: int
    d: np.ndarray  # (40, m)
    u: np.ndarray  # (40, rank, m)
    v: np.ndarray  # (40, rank, m)


@dataclass
class ToeplitzRep:
    nx: int
    ny: int
    m: int
    generators: np.ndarray  # (nb, m, m) column-major blocks, raw layout of gen.blocks_raw
    correction: Correction | None = None
    margin: "Margin | None" = None
    # "sparse": the reference's canonical half (nx*ny + (nx-1)*(ny-1) blocks,
    # A(-s) = A(s)^T); "full": every shift, (2ny-1)*(2nx-1) blocks, i = 1-ny
    # .. ny-1 outer, j = 1-nx .. nx-1 inner (non-reciprocal operators).
    layout: str = "sparse"

    @classmethod
    def synthetic(cls, cfg) -> "ToeplitzRep":
        from . import gen
        blk = gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed)
        corr = None
        if cfg.rank >= 0 and cfg.scale > 0:
            d, u, v = gen.correction(cfg.m, cfg.rank, cfg.seed, cfg.scale)
            corr = Correction(cfg.rank, d, u, v)
        return cls(cfg.nx, cfg.ny, cfg.m, blk, corr)

    def elementEdges(self) -> int:  # toeplitz.hpp:98
        return self.nx * self.ny * self.m


@dataclass
class Margin:
    """Margin coupling B / B^T / C (ToeplitzRep::bSideGen, bRowGen, bCorner
    and the margin x margin blocks, toeplitz.hpp:76-95; layouts in
    include/tbt_gen.h). e: edges per part of components 1..9 (e[4] = m)."""
    e: list
    bside: np.ndarray
    brow: np.ndarray
    bcorner: np.ndarray
    c: np.ndarray

    def size(self, nx: int, ny: int) -> int:  # ToeplitzRep::marginEdges, toeplitz.hpp:99-102
        e = self.e
        return ny * (e[1] + e[7]) + nx * (e[5] + e[3]) + e[2] + e[8] + e[0] + e[6]


@dataclass
class DenseMargin:
    """Margin coupling of a SemiSparse representation (ToeplitzRep::bFull,
    cFull, toeplitz.hpp:90-93): B (nM x nA) and C (nM x nM) as dense
    matrices, flattened column-major. e as in Margin."""
    e: list
    b_full: np.ndarray
    c: np.ndarray

    def size(self, nx: int, ny: int) -> int:
        e = self.e
        return ny * (e[1] + e[7]) + nx * (e[5] + e[3]) + e[2] + e[8] + e[0] + e[6]


def generators_from_level1(nx: int, ny: int, m: int, a_level1) -> np.ndarray:
    """Canonical Sparse-order generator blocks (gen.blocks_raw layout) read
    out of SemiSparse first-level blocks: shift (i, j) is block
    (max(j, 0), max(-j, 0)) of aLevel1[i] (aEntry, linsolve.cpp:220-224)."""
    blocks = []
    for i in range(ny):
        a1 = np.asarray(a_level1[i])
        for j in range(0 if i == 0 else 1 - nx, nx):
            r0, c0 = max(j, 0) * m, max(-j, 0) * m
            blocks.append(a1[r0:r0 + m, c0:c0 + m].T)  # raw [b][a] = column-major (a, b)
    return np.ascontiguousarray(np.stack(blocks), dtype=np.complex128)


@dataclass
class SolverOptions:  # linsolve.hpp:47-53
    tol: float = 1e-8
    maxIter: int = 2000
    restart: int = 60
    precondition: bool = True
    threads: int = 1  # accepted for API parity; columns run in lockstep on the GPU
    orthog: int = 1   # 0: MGS projection sweep; 1: low-synchronisation MGS (same coefficients)


@dataclass
class SolveResult:  # linsolve.hpp:40-45
    current: np.ndarray
    residual: list
    iterations: list
    solver: str = "gmres"
    converged: list = field(default_factory=list)
    history: list = field(default_factory=list)
    matvecs: int = 0


def _as_cols(x: np.ndarray) -> tuple[np.ndarray, int, bool]:
    x = np.asarray(x, dtype=np.complex128)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    return np.asfortranarray(x), x.shape[1], vec


def _generator_key(generators) -> bytes:
    """32-byte digest naming a generator set (tbt_set_cache_key): BLAKE2b over
    the BLAKE2b digests of 64 MiB slices, the slices hashed on a thread pool
    (hashlib releases the GIL) -- one serial BLAKE2b pass over C4's 2.1 GB of
    blocks took 2 s, ten times the whole K1 setup it guards."""
    import hashlib
    import os
    from concurrent.futures import ThreadPoolExecutor
    raw = np.ascontiguousarray(generators).view(np.uint8).ravel()
    step = 64 << 20
    parts = [raw[i:i + step] for i in range(0, raw.size, step)] or [raw]
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1, len(parts))) as ex:
        digests = list(ex.map(lambda b: hashlib.blake2b(b, digest_size=32).digest(), parts))
    top = hashlib.blake2b(digest_size=32)
    top.update(str(tuple(np.shape(generators))).encode())
    for d in digests:
        top.update(d)
    return top.digest()


class ToeplitzMatvec:
    """FFT-accelerated application of Z^part (linsolve.hpp:59-77) on a B200."""

    def __init__(self, rep: ToeplitzRep, max_nrhs: int = 1, device: int = 0, embed: str = "pow2",
                 dist: tuple | None = None, spectra_cache: str | None = None):
        """embed: "pow2" (the reference's nextPow2 embedding) or "smooth"
        (smallest 2^a 3^b length per level, mixed-radix transforms).
        dist: (nranks, rank, nccl_unique_id_bytes) to shard the operator over
        one process per GPU (see dist_unique_id / init_from_torch); apply /
        applyA / diagonal then work on this rank's element-row slab.
        (nranks, rank, group_id, "loopback") runs rank `rank` of the same
        sharded operator in this process (tbt_dist_init_loopback; see
        loopback_group_id): every rank's calls must then be issued
        concurrently, one host thread per rank.
        spectra_cache: a TBTS1 file; loaded instead of K1 when it exists,
        written after K1 otherwise (row f3). The cache is keyed by a BLAKE2b
        digest of rep.generators (tbt_set_cache_key): a file written for
        other generators of the same shape is rejected (UserError). A rep
        without generators (shape only) loads any cache of its shape."""
        self.rep = rep
        self._h = C.c_void_p()
        if embed not in ("pow2", "smooth"):
            raise UserError(f"embed must be 'pow2' or 'smooth', got {embed!r}")
        desc = TbtDesc(rep.nx, rep.ny, rep.m, max_nrhs, device, 1 if embed == "smooth" else 0)
        _check(lib().tbt_create(C.byref(desc), C.byref(self._h)))
        import os
        cached = spectra_cache is not None and os.path.exists(spectra_cache)
        if spectra_cache is not None and rep.generators.size:
            key = _generator_key(rep.generators)
            _check(lib().tbt_set_cache_key(self._h, key, len(key)))
        if not cached:
            gen = np.ascontiguousarray(rep.generators, dtype=np.complex128)
            setg = lib().tbt_set_generators_full if rep.layout == "full" else lib().tbt_set_generators
            _check(setg(self._h, gen.ctypes.data_as(dp), gen.shape[0]))
        if rep.correction is not None:
            c = rep.correction
            d = np.ascontiguousarray(c.d)
            u = np.ascontiguousarray(c.u) if c.rank > 0 else None
            v = np.ascontiguousarray(c.v) if c.rank > 0 else None
            _check(lib().tbt_set_correction(self._h, c.rank, d.ctypes.data_as(dp),
                                            u.ctypes.data_as(dp) if u is not None else None,
                                            v.ctypes.data_as(dp) if v is not None else None))
        if isinstance(rep.margin, DenseMargin):
            mg = rep.margin
            e = np.ascontiguousarray(mg.e, dtype=np.int32)
            b = np.ascontiguousarray(mg.b_full, dtype=np.complex128)
            cm = np.ascontiguousarray(mg.c, dtype=np.complex128)
            b = b if b.size else np.zeros(1, np.complex128)
            cm = cm if cm.size else np.zeros(1, np.complex128)
            _check(lib().tbt_set_margin_dense(self._h, e.ctypes.data_as(C.POINTER(C.c_int)), b.ctypes.data_as(dp),
                                              cm.ctypes.data_as(dp)))
        elif rep.margin is not None:
            mg = rep.margin
            e = np.ascontiguousarray(mg.e, dtype=np.int32)
            arrs = [np.ascontiguousarray(a, dtype=np.complex128) for a in (mg.bside, mg.brow, mg.bcorner, mg.c)]
            arrs = [a if a.size else np.zeros(1, np.complex128) for a in arrs]
            _check(lib().tbt_set_margin(self._h, e.ctypes.data_as(C.POINTER(C.c_int)),
                                        *[a.ctypes.data_as(dp) for a in arrs]))
        if dist is not None:
            nranks, rank, uid = dist[:3]
            transport = dist[3] if len(dist) > 3 else "nccl"
            if transport not in ("nccl", "loopback"):
                raise UserError(f"transport must be 'nccl' or 'loopback', got {transport!r}")
            init = lib().tbt_dist_init_loopback if transport == "loopback" else lib().tbt_dist_init
            _check(init(self._h, int(nranks), int(rank), bytes(uid)))
        if cached:
            _check(lib().tbt_load_spectra(self._h, spectra_cache.encode()))
        else:
            _check(lib().tbt_precompute(self._h))
            if spectra_cache is not None:
                _check(lib().tbt_save_spectra(self._h, spectra_cache.encode()))
        self.max_nrhs = max_nrhs

    @classmethod
    def from_ztoe1(cls, path: str, max_nrhs: int = 1, device: int = 0, embed: str = "pow2") -> "ToeplitzMatvec":
        """Operator from a reference ZTOE1 block cache (saveBlockCache,
        toeplitz.cpp:700-743; Sparse mode), precomputed (row f3)."""
        nx, ny = C.c_int(), C.c_int()
        e = (C.c_int * 9)()
        _check(lib().tbt_ztoe1_dims(path.encode(), C.byref(nx), C.byref(ny), e))
        self = cls.__new__(cls)
        self.rep = ToeplitzRep(nx.value, ny.value, e[4], np.empty((0, e[4], e[4]), np.complex128))
        self._h = C.c_void_p()
        _check(lib().tbt_load_ztoe1(path.encode(), max_nrhs, device, 1 if embed == "smooth" else 0,
                                    C.byref(self._h)))
        self.max_nrhs = max_nrhs
        return self

    def close(self) -> None:
        if self._h:
            lib().tbt_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- reference methods -------------------------------------------------
    def sizeA(self) -> int:
        """Unknowns held by this process (the row slab when distributed)."""
        r0, r1 = self.rows()
        return (r1 - r0) * self.rep.nx * self.rep.m

    def rows(self) -> tuple[int, int]:
        """Element rows [begin, end) this process owns (all rows unless distributed)."""
        a, b = C.c_int(), C.c_int()
        _check(lib().tbt_dist_rows(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def sizeM(self) -> int:
        """Margin unknowns (ToeplitzMatvec::sizeM, linsolve.hpp:72); 0 without margin data."""
        return int(lib().tbt_size_m(self._h))

    def size(self) -> int:
        """Unknowns of apply / diagonal / gmres: sizeA() + sizeM()."""
        return self.sizeA() + self.sizeM()

    def _apply(self, fn, x, n: int, n_out: int | None = None):
        xc, k, vec = _as_cols(x)
        if xc.shape[0] != n:
            raise UserError(f"matvec: vector length {xc.shape[0]} does not match system size {n}")
        y = np.empty((n if n_out is None else n_out, k), dtype=np.complex128, order="F")
        _check(fn(self._h, xc.ctypes.data, y.ctypes.data, k, TBT_HOST))
        return y[:, 0] if vec else y

    def apply(self, x):
        return self._apply(lib().tbt_apply, x, self.size())

    def applyA(self, x):
        return self._apply(lib().tbt_apply_a, x, self.sizeA())

    def apply_many(self, X) -> np.ndarray:
        """Z x_i for a batch of independent vectors, X of shape (count, n)
        (one vector per row); host copies overlap the applies
        (tbt_apply_many). Pageable numpy memory serialises the copies: pass
        pinned buffers to apply_many_ptr for the overlapped stream."""
        X = np.ascontiguousarray(X, dtype=np.complex128)
        if X.ndim != 2 or X.shape[1] != self.size():
            raise ValueError(f"apply_many: X must have shape (count, {self.size()})")
        Y = np.empty_like(X)
        _check(lib().tbt_apply_many(self._h, X.ctypes.data, Y.ctypes.data, X.shape[0]))
        return Y

    def apply_many_ptr(self, x_ptr: int, y_ptr: int, count: int) -> None:
        """tbt_apply_many on host pointers (e.g. pinned torch tensors)."""
        _check(lib().tbt_apply_many(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), count))

    def applyB(self, xA):
        """yM = B xA (linsolve.hpp:66, linsolve.cpp:292-314)."""
        return self._apply(lib().tbt_apply_b, xA, self.sizeA(), self.sizeM())

    def applyBT(self, xM):
        """yA = B^T xM (linsolve.hpp:67, linsolve.cpp:316-334)."""
        return self._apply(lib().tbt_apply_bt, xM, self.sizeM(), self.sizeA())

    def applyC(self, xM):
        """yM = C xM (linsolve.hpp:68, linsolve.cpp:336-349)."""
        return self._apply(lib().tbt_apply_c, xM, self.sizeM(), self.sizeM())

    def diagonal(self) -> np.ndarray:
        d = np.empty(self.size(), dtype=np.complex128)
        _check(lib().tbt_diagonal(self._h, d.ctypes.data_as(dp)))
        return d

    # -- device-pointer entry points (bench / torch interop) ----------------
    def apply_device(self, x_ptr: int, y_ptr: int, nrhs: int = 1, a_only: bool = False) -> None:
        fn = lib().tbt_apply_a if a_only else lib().tbt_apply
        _check(fn(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), nrhs, TBT_DEVICE))

    def set_stream(self, stream_ptr: int | None) -> None:
        _check(lib().tbt_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def stream(self) -> int:
        return int(lib().tbt_get_stream(self._h) or 0)

    def info(self) -> TbtInfo:
        inf = TbtInfo()
        _check(lib().tbt_get_info(self._h, C.byref(inf)))
        return inf

    def spectrum_bin(self, f: int) -> np.ndarray:
        out = np.empty((self.rep.m, self.rep.m), dtype=np.complex128)
        _check(lib().tbt_get_spectrum_bin(self._h, f, out.ctypes.data_as(dp)))
        return out

    def set_timing(self, on: bool) -> None:
        _check(lib().tbt_set_timing(self._h, 1 if on else 0))

    def timing_read(self) -> tuple[float, int]:
        tot, cnt = C.c_double(), C.c_int()
        _check(lib().tbt_timing_read(self._h, C.byref(tot), C.byref(cnt)))
        return tot.value, cnt.value

    def phase_times(self, on: bool = True):
        out = (C.c_double * 13)()
        _check(lib().tbt_phase_times(self._h, 1 if on else 0, out))
        return list(out)

    def cta_trace(self):
        """Per-CTA event times of the last 8 persistent applies (TBT_CTATRACE=1):
        (launches, array [8 slots][16 events][256 CTAs] of uint64)."""
        import numpy as np
        n = 8 * 16 * 256
        buf = (C.c_ulonglong * n)()
        cnt = C.c_longlong()
        _check(lib().tbt_cta_trace(self._h, buf, n, C.byref(cnt)))
        return cnt.value, np.frombuffer(buf, dtype=np.uint64).reshape(8, 16, 256).copy()

    def bench_apply(self, x_ptr: int, y_ptr: int, iters: int, use_graph: bool = True):
        ms, bms = C.c_double(), C.c_double()
        _check(lib().tbt_bench_apply(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), 1, iters,
                                     1 if use_graph else 0, C.byref(ms), C.byref(bms)))
        return ms.value, bms.value

    def gmres(self, b, opt: SolverOptions, use_a_only: bool = False, hist_cap: int = 4096,
              raise_on_fail: bool = True, where: int = TBT_HOST, b_ptr: int = 0, x_ptr: int = 0,
              nrhs: int | None = None) -> SolveResult:
        if where == TBT_HOST:
            bc, k, vec = _as_cols(b)
            x = np.empty_like(bc, order="F")
            bp, xp = bc.ctypes.data, x.ctypes.data
        else:
            k, vec, x = int(nrhs), False, None
            bp, xp = b_ptr, x_ptr
        its = np.zeros(k, dtype=np.int32)
        res = np.zeros(k, dtype=np.float64)
        conv = np.zeros(k, dtype=np.int32)
        hlen = np.zeros(k, dtype=np.int32)
        hist = np.zeros((k, max(hist_cap, 1), 2), dtype=np.float64)
        st = TbtGmresStats(its.ctypes.data_as(C.POINTER(C.c_int)), res.ctypes.data_as(dp),
                           conv.ctypes.data_as(C.POINTER(C.c_int)), hist.ctypes.data_as(dp),
                           hlen.ctypes.data_as(C.POINTER(C.c_int)), 0)
        o = TbtGmresOpts(opt.tol, opt.maxIter, opt.restart, 1 if opt.precondition else 0,
                         1 if use_a_only else 0, hist_cap, opt.orthog)
        status = lib().tbt_gmres(self._h, C.c_void_p(bp), C.c_void_p(xp), k, C.byref(o), C.byref(st), where)
        if status not in (_lib.TBT_OK, _lib.TBT_NUMERIC_ERROR) or (status != _lib.TBT_OK and raise_on_fail):
            _check(status)
        histories = [hist[c, :min(int(hlen[c]), hist_cap)].copy() for c in range(k)]
        cur = None if x is None else (x[:, 0] if vec else x)
        return SolveResult(cur, res.tolist(), its.tolist(), "gmres", conv.tolist(), histories, st.matvecs)

    def schur_solve(self, b, opt: SolverOptions) -> SolveResult:
        """schurSolve (linsolve.cpp:595-682) on the device: b is (sizeA + sizeM)
        x p with zero margin rows. Raises UserError / NumericError like the
        reference (inner solve not converged, singular Schur complement)."""
        bc, k, vec = _as_cols(b)
        if bc.shape[0] != self.size():
            raise UserError(f"schurSolve: excitation size mismatch ({bc.shape[0]} vs {self.size()})")
        x = np.empty_like(bc, order="F")
        its = np.zeros(k, dtype=np.int32)
        res = np.zeros(k, dtype=np.float64)
        conv = np.zeros(k, dtype=np.int32)
        hlen = np.zeros(k, dtype=np.int32)
        st = TbtGmresStats(its.ctypes.data_as(C.POINTER(C.c_int)), res.ctypes.data_as(dp),
                           conv.ctypes.data_as(C.POINTER(C.c_int)), None, hlen.ctypes.data_as(C.POINTER(C.c_int)), 0)
        o = TbtGmresOpts(opt.tol, opt.maxIter, opt.restart, 1 if opt.precondition else 0, 1, 0, opt.orthog)
        _check(lib().tbt_schur_solve(self._h, C.c_void_p(bc.ctypes.data), C.c_void_p(x.ctypes.data), k, C.byref(o),
                                     C.byref(st), TBT_HOST))
        return SolveResult(x[:, 0] if vec else x, res.tolist(), its.tolist(), "schur", conv.tolist(), [], 0)



# -- row f4: contractions on solved currents (postproc.cpp) ----------------
def port_network(op: "ToeplitzMatvec", current, feed_rows, edge_len: float, z0) -> dict:
    """portNetwork (postproc.cpp:186-230) on the device: Y = I/len^2 from the
    port rows of the solution, Z = Y^-1, power-wave S. dict(y, z, s)."""
    cur = np.asfortranarray(current, dtype=np.complex128)
    p = cur.shape[1]
    feed = np.ascontiguousarray(feed_rows, dtype=np.int64)
    z0 = np.ascontiguousarray(z0, dtype=np.float64)
    if feed.size != p or z0.size != p:
        raise UserError("portNetwork: need one feed row and one Z0 per port")
    out = [np.empty((p, p), np.complex128, order="F") for _ in range(3)]
    _check(lib().tbt_port_network(op._h, cur.ctypes.data_as(dp), cur.shape[0], p,
                                  feed.ctypes.data_as(C.POINTER(C.c_longlong)), float(edge_len), z0.ctypes.data_as(dp),
                                  *[o.ctypes.data_as(dp) for o in out], TBT_HOST))
    return dict(y=out[0], z=out[1], s=out[2])


def tarc(s, a) -> float:
    """Total active reflection coefficient |S a| / |a| (postproc.cpp:232-236)."""
    a = np.asarray(a, dtype=np.complex128)
    an = np.linalg.norm(a)
    if an == 0.0:
        raise UserError("tarc: zero excitation")
    return float(np.linalg.norm(np.asarray(s) @ a) / an)


def array_farfield(op: "ToeplitzMatvec", tensors, e, dirs, dx: float, dy: float, k: float, eta: float, current,
                   weights):
    """arrayFarfield (postproc.cpp:134-170) for the columns of current @ weights
    on the device; weights = identity gives embeddedElementPatterns
    (:172-184). tensors[c] = (co, cx), each ndir x e[c], or None. Returns
    (co, cx), ndir x q."""
    ea = np.ascontiguousarray(e, dtype=np.int32)
    keep = []
    pco, pcx = (dp * 9)(), (dp * 9)()
    for c in range(9):
        if ea[c] == 0 or tensors[c] is None:
            pco[c] = pcx[c] = None
            continue
        a = np.asfortranarray(tensors[c][0], dtype=np.complex128)
        b = np.asfortranarray(tensors[c][1], dtype=np.complex128)
        keep += [a, b]
        pco[c], pcx[c] = a.ctypes.data_as(dp), b.ctypes.data_as(dp)
    d = np.ascontiguousarray(dirs, dtype=np.float64)
    cur = np.asfortranarray(current, dtype=np.complex128)
    W = np.asarray(weights, dtype=np.complex128)
    W = np.asfortranarray(W[:, None] if W.ndim == 1 else W)
    ndir, q = d.shape[0], W.shape[1]
    co = np.empty((ndir, q), np.complex128, order="F")
    cx = np.empty_like(co)
    _check(lib().tbt_array_farfield(op._h, pco, pcx, ea.ctypes.data_as(C.POINTER(C.c_int)), ndir, d.ctypes.data_as(dp),
                                    dx, dy, k, eta, cur.ctypes.data_as(dp), cur.shape[1], W.ctypes.data_as(dp), q,
                                    co.ctypes.data_as(dp), cx.ctypes.data_as(dp), TBT_HOST))
    return co, cx


def read_ztoe1(path: str) -> ToeplitzRep:
    """A reference ZTOE1 block cache as a ToeplitzRep with its margin data
    (host-side parse, csrc/io.cu; row f3): Sparse caches give a Margin,
    SemiSparse caches a DenseMargin (generators read out of aLevel1)."""
    from . import gen as _gen
    nx, ny = C.c_int(), C.c_int()
    e = (C.c_int * 9)()
    _check(lib().tbt_ztoe1_dims(path.encode(), C.byref(nx), C.byref(ny), e))
    nx, ny, ev = nx.value, ny.value, [int(v) for v in e]
    m = ev[4]
    nb = _gen.num_blocks(nx, ny)
    g = np.empty((nb, m, m), np.complex128)
    mode = C.c_int()
    _check(lib().tbt_ztoe1_mode(path.encode(), C.byref(mode)))
    if mode.value == 1:
        dm = DenseMargin(ev, np.empty(0, np.complex128), np.empty(0, np.complex128))
        nA = nx * ny * m
        nM = dm.size(nx, ny)
        bf = np.empty(max(nM * nA, 1), np.complex128)
        cf = np.empty(max(nM * nM, 1), np.complex128)
        _check(lib().tbt_ztoe1_read_dense(path.encode(), g.ctypes.data_as(dp), bf.ctypes.data_as(dp),
                                          cf.ctypes.data_as(dp)))
        margin = DenseMargin(ev, bf[:nM * nA], cf[:nM * nM]) if nM else None
        return ToeplitzRep(nx, ny, m, g, None, margin)
    ea = np.ascontiguousarray(ev, dtype=np.int32)
    ns, nr, nc = C.c_longlong(), C.c_longlong(), C.c_longlong()
    nM = int(lib().tbtgen_margin_lengths(nx, ny, ea.ctypes.data_as(C.POINTER(C.c_int)), C.byref(ns), C.byref(nr),
                                         C.byref(nc)))
    arrs = [np.empty(max(n, 1), np.complex128) for n in (ns.value, nr.value, nc.value, nM * nM)]
    _check(lib().tbt_ztoe1_read(path.encode(), g.ctypes.data_as(dp), *[a.ctypes.data_as(dp) for a in arrs]))
    margin = None
    if nM > 0:
        margin = Margin(ev, arrs[0][:ns.value], arrs[1][:nr.value], arrs[2][:nc.value], arrs[3][:nM * nM])
    return ToeplitzRep(nx, ny, m, g, None, margin)


def dist_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for tbt_dist_init (call on rank 0)."""
    buf = C.create_string_buffer(128)
    _check(lib().tbt_dist_unique_id(buf))
    return buf.raw


def loopback_group_id() -> bytes:
    """A fresh 128-byte id naming one in-process loopback group."""
    import os
    return os.urandom(128)


def dist_plan(ny: int, L0: int, nranks: int, rank: int):
    """(row_begin, row_end, columns) of `rank` in the multi-GPU partition."""
    rb, re_, nc = C.c_int(), C.c_int(), C.c_int()
    cols = (C.c_int * max(L0, 1))()
    _check(lib().tbt_dist_plan(ny, L0, nranks, rank, C.byref(rb), C.byref(re_), C.byref(nc), cols))
    return rb.value, re_.value, [cols[k] for k in range(nc.value)]


def init_from_torch(group=None) -> tuple:
    """(nranks, rank, uid) for ToeplitzMatvec(dist=...) from an initialised
    torch.distributed process group (rank 0 makes the id, all receive it)."""
    import torch.distributed as tdist
    rank, world = tdist.get_rank(group), tdist.get_world_size(group)
    obj = [dist_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0, group=group)
    return world, rank, obj[0]


def toeplitz_matvec(rep: ToeplitzRep, x) -> np.ndarray:
    """One-shot wrapper (linsolve.hpp:80-81)."""
    op = ToeplitzMatvec(rep)
    try:
        return op.apply(x)
    finally:
        op.close()


def schur_solve(rep: ToeplitzRep, V, opt: SolverOptions | None = None) -> SolveResult:
    """schurSolve (linsolve.hpp:93-95) through the device operator."""
    opt = opt or SolverOptions()
    k = 1 if np.ndim(V) == 1 else np.shape(V)[1]
    op = ToeplitzMatvec(rep, max_nrhs=max(1, min(k + (rep.margin.size(rep.nx, rep.ny) if rep.margin else 0), 64)))
    try:
        return op.schur_solve(V, opt)
    finally:
        op.close()


def iterative_solve(rep: ToeplitzRep, V, opt: SolverOptions | None = None) -> SolveResult:
    """iterativeSolve (linsolve.cpp:551-593): restarted GMRES per column,
    Jacobi on by default; raises NumericError if a column does not converge."""
    opt = opt or SolverOptions()
    Vc, k, _ = _as_cols(V)
    op = ToeplitzMatvec(rep, max_nrhs=k)
    try:
        if Vc.shape[0] != op.sizeA():
            raise UserError("iterativeSolve: excitation size mismatch")
        return op.gmres(V, opt)
    finally:
        op.close()
