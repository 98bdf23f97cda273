"""CPU oracle (TEST INFRASTRUCTURE ONLY).

ctypes binding of oracle/liboracle.so, a C++ restatement of the
reference's matvec / GMRES (see oracle/oracle.h for the file:line map), and
of oracle/_ref/libref_fft.so, the reference's own fftInPlace compiled from
/root/reference/proj/src/fft.cpp. Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import this package, as the checker or the timed CPU
baseline; the product path (paper_2506_04710_b200 / libtbt.so) never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_FFT_SO = HERE / "_ref" / "libref_fft.so"

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_SO))
        L.orc_next_pow2.restype = C.c_size_t
        L.orc_next_pow2.argtypes = [C.c_size_t]
        L.orc_fft.restype = C.c_int
        L.orc_fft.argtypes = [dp, C.c_size_t, C.c_int]
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        L.orc_create_full.restype = C.c_void_p
        L.orc_create_full.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        L.orc_destroy.restype = None
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_precompute.argtypes = [C.c_void_p, C.c_int]
        L.orc_ahat.argtypes = [C.c_void_p, dp]
        L.orc_bins.restype = C.c_longlong
        L.orc_bins.argtypes = [C.c_void_p]
        L.orc_set_correction.argtypes = [C.c_void_p, C.c_int, dp, dp, dp]
        L.orc_set_margin.argtypes = [C.c_void_p, ip, dp, dp, dp, dp]
        L.orc_set_margin_dense.argtypes = [C.c_void_p, ip, dp, dp]
        L.orc_size.restype = C.c_longlong
        L.orc_size.argtypes = [C.c_void_p]
        L.orc_schur.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                ip, dp, C.c_char_p, C.c_int]
        L.orc_port_network.argtypes = [dp, C.c_longlong, C.c_int, C.POINTER(C.c_longlong), C.c_double, dp, dp, dp,
                                       dp]
        L.orc_array_farfield.argtypes = [C.c_int, C.c_int, ip, C.POINTER(dp), C.POINTER(dp), C.c_int, dp, C.c_double,
                                         C.c_double, C.c_double, C.c_double, dp, C.c_int, dp, C.c_int, dp, dp]
        L.orc_apply_a.argtypes = [C.c_void_p, dp, dp]
        L.orc_apply.argtypes = [C.c_void_p, dp, dp]
        L.orc_apply_cols.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_int, C.c_int]
        L.orc_apply_rows.argtypes = [C.c_void_p, dp, C.POINTER(C.c_longlong), C.c_longlong, dp]
        L.orc_dense.argtypes = [C.c_void_p, dp]
        L.orc_sampled_apply.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(dp), C.POINTER(dp), dp, dp, dp,
                                        dp, C.c_int]
        L.orc_diagonal.argtypes = [C.c_void_p, dp]
        L.orc_gmres.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.c_int, ip, dp, ip, dp, C.c_int, ip]
        _lib = L
    return _lib


def ref_lib() -> C.CDLL | None:
    """The reference's own fft.cpp (None when oracle/_ref was not built)."""
    global _ref
    if _ref is None and REF_FFT_SO.exists():
        L = C.CDLL(str(REF_FFT_SO))
        L.ref_next_pow2.restype = C.c_size_t
        L.ref_next_pow2.argtypes = [C.c_size_t]
        L.ref_fft.restype = C.c_int
        L.ref_fft.argtypes = [dp, C.c_size_t, C.c_int]
        _ref = L
    return _ref


def bind_inputs() -> None:
    """Routes paper_2506_04710_b200.gen (the seeded inputs of tbt_gen.h) to
    liboracle.so's copy of csrc/gen.cpp, so a CPU-only process (bench.py
    --impl reference) never maps the product library."""
    from paper_2506_04710_b200 import gen
    gen.bind(lib())


def product_mapped() -> bool:
    """True when libtbt.so is mapped into this process."""
    try:
        return "libtbt.so" in open("/proc/self/maps").read()
    except OSError:
        return False


def _p(a: np.ndarray):
    return a.ctypes.data_as(dp)


def fft(a: np.ndarray, inverse: bool = False) -> np.ndarray:
    out = np.array(a, dtype=np.complex128, copy=True)
    if lib().orc_fft(_p(out), out.size, 1 if inverse else 0):
        raise ValueError("fftInPlace: length must be a power of two")
    return out


def ref_fft(a: np.ndarray, inverse: bool = False) -> np.ndarray:
    out = np.array(a, dtype=np.complex128, copy=True)
    if ref_lib().ref_fft(_p(out), out.size, 1 if inverse else 0):
        raise ValueError("fftInPlace: length must be a power of two")
    return out


class Oracle:
    """Restated ToeplitzMatvec + gmres over canonical Sparse generators."""

    def __init__(self, nx, ny, m, generators_raw: np.ndarray, correction=None, precompute=True,
                 nthreads: int = 0, margin=None, layout: str = "sparse"):
        self.nx, self.ny, self.m = nx, ny, m
        self.nA = self.n = nx * ny * m
        g = np.ascontiguousarray(generators_raw, dtype=np.complex128)
        create = lib().orc_create_full if layout == "full" else lib().orc_create
        self._h = create(nx, ny, m, _p(g))
        if not self._h:
            raise ValueError("orc_create failed")
        if correction is not None:
            rank, d, u, v = correction
            d = np.ascontiguousarray(d)
            u = np.ascontiguousarray(u) if rank > 0 else np.zeros(1, np.complex128)
            v = np.ascontiguousarray(v) if rank > 0 else np.zeros(1, np.complex128)
            lib().orc_set_correction(self._h, rank, _p(d), _p(u), _p(v))
        if margin is not None and hasattr(margin, "b_full"):  # DenseMargin (SemiSparse)
            e = np.ascontiguousarray(margin.e, dtype=np.int32)
            arrs = [np.ascontiguousarray(a, dtype=np.complex128) for a in (margin.b_full, margin.c)]
            arrs = [a if a.size else np.zeros(1, np.complex128) for a in arrs]
            if lib().orc_set_margin_dense(self._h, e.ctypes.data_as(ip), *[_p(a) for a in arrs]):
                raise ValueError("orc_set_margin_dense failed")
            self._margin_keep = arrs
            self.n = int(lib().orc_size(self._h))
        elif margin is not None:
            e = np.ascontiguousarray(margin.e, dtype=np.int32)
            arrs = [np.ascontiguousarray(a, dtype=np.complex128) for a in
                    (margin.bside, margin.brow, margin.bcorner, margin.c)]
            arrs = [a if a.size else np.zeros(1, np.complex128) for a in arrs]
            if lib().orc_set_margin(self._h, e.ctypes.data_as(ip), *[_p(a) for a in arrs]):
                raise ValueError("orc_set_margin failed")
            self._margin_keep = arrs
            self.n = int(lib().orc_size(self._h))
        if precompute:
            self.precompute(nthreads)

    @classmethod
    def from_rep(cls, rep, precompute=True, nthreads: int = 0):
        corr = None
        if rep.correction is not None:
            c = rep.correction
            corr = (c.rank, c.d, c.u, c.v)
        return cls(rep.nx, rep.ny, rep.m, rep.generators, corr, precompute, nthreads,
                   getattr(rep, "margin", None), getattr(rep, "layout", "sparse"))

    def precompute(self, nthreads: int = 0):
        lib().orc_precompute(self._h, nthreads)

    def close(self):
        if self._h:
            lib().orc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def bins(self) -> int:
        return int(lib().orc_bins(self._h))

    def ahat(self) -> np.ndarray:
        """Reference layout [(m*e5+n)*L + f] reshaped to (m, m, L)."""
        out = np.empty((self.m, self.m, self.bins), dtype=np.complex128)
        if lib().orc_ahat(self._h, _p(out)):
            raise RuntimeError("no spectra")
        return out

    def _vec(self, fn, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.empty_like(x)
        if fn(self._h, _p(x), _p(y)):
            raise RuntimeError("oracle apply failed")
        return y

    def apply(self, x):
        return self._vec(lib().orc_apply, x)

    def applyA(self, x):
        return self._vec(lib().orc_apply_a, x)

    def apply_cols(self, X, nthreads=0, a_only=False):
        X = np.asfortranarray(X, dtype=np.complex128)
        Y = np.empty_like(X, order="F")
        if lib().orc_apply_cols(self._h, _p(X), _p(Y), X.shape[1], nthreads, 1 if a_only else 0):
            raise RuntimeError("orc_apply_cols failed")
        return Y

    def apply_rows(self, x, elems):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        el = np.ascontiguousarray(elems, dtype=np.int64)
        y = np.empty((len(el), self.m), dtype=np.complex128)
        if lib().orc_apply_rows(self._h, _p(x), el.ctypes.data_as(C.POINTER(C.c_longlong)), len(el), _p(y)):
            raise RuntimeError("orc_apply_rows failed")
        return y

    def dense(self):
        """Dense A (+ correction), nA x nA (margin excluded)."""
        z = np.empty((self.nA, self.nA), dtype=np.complex128, order="F")
        lib().orc_dense(self._h, _p(z))
        return z

    def diagonal(self):
        d = np.empty(self.n, dtype=np.complex128)
        lib().orc_diagonal(self._h, _p(d))
        return d

    def schur(self, b, tol=1e-8, max_iter=2000, restart=60, precondition=True, nthreads=1):
        """schurSolve restated: dict(x, iterations, residual) or raises
        ValueError (user error) / ArithmeticError (numeric)."""
        b = np.asarray(b, dtype=np.complex128)
        vec = b.ndim == 1
        bc = np.asfortranarray(b[:, None] if vec else b)
        k = bc.shape[1]
        x = np.empty_like(bc, order="F")
        its = np.zeros(k, np.int32)
        res = np.zeros(k, np.float64)
        err = C.create_string_buffer(512)
        st = lib().orc_schur(self._h, _p(bc), _p(x), k, tol, max_iter, restart, 1 if precondition else 0, nthreads,
                             its.ctypes.data_as(ip), _p(res), err, 512)
        if st == 1:
            raise ValueError(err.value.decode())
        if st == 2:
            raise ArithmeticError(err.value.decode())
        return dict(x=x[:, 0] if vec else x, iterations=its.tolist(), residual=res.tolist())

    def gmres(self, b, tol=1e-8, max_iter=2000, restart=60, precondition=True, use_a_only=False,
              nthreads=1, hist_cap=4096):
        b = np.asarray(b, dtype=np.complex128)
        vec = b.ndim == 1
        bc = np.asfortranarray(b[:, None] if vec else b)
        k = bc.shape[1]
        x = np.empty_like(bc, order="F")
        its = np.zeros(k, np.int32)
        res = np.zeros(k, np.float64)
        conv = np.zeros(k, np.int32)
        hist = np.zeros((k, hist_cap, 2), np.float64)
        hlen = np.zeros(k, np.int32)
        lib().orc_gmres(self._h, _p(bc), _p(x), k, tol, max_iter, restart, 1 if precondition else 0,
                        1 if use_a_only else 0, nthreads, its.ctypes.data_as(ip), _p(res),
                        conv.ctypes.data_as(ip), _p(hist), hist_cap, hlen.ctypes.data_as(ip))
        hists = [hist[c, :min(int(hlen[c]), hist_cap)].copy() for c in range(k)]
        return dict(x=x[:, 0] if vec else x, iterations=its.tolist(), residual=res.tolist(),
                    converged=conv.tolist(), history=hists)


def sampled_apply(nx, ny, m, seed, rows, x, nthreads=0):
    """Bounded sample of the reference's applyA (orc_sampled_apply): output
    rows `rows` (basis indices) of every element, plus the timed forward
    section and the timed per-row section (single thread). Needs only
    row / column `a` of each canonical block (gen.block_lines), so it runs at
    C5 where the spectra (38.65 GB) do not fit host memory."""
    from paper_2506_04710_b200 import gen
    lines = [gen.block_lines(nx, ny, m, seed, int(a), nthreads) for a in rows]
    pr = (dp * len(rows))(*[_p(r) for r, _ in lines])
    pc = (dp * len(rows))(*[_p(c) for _, c in lines])
    x = np.ascontiguousarray(x, dtype=np.complex128)
    y = np.empty((len(rows), nx * ny), np.complex128)
    tf, tr = C.c_double(), C.c_double()
    if lib().orc_sampled_apply(nx, ny, m, len(rows), pr, pc, _p(x), _p(y), C.byref(tf), C.byref(tr), nthreads):
        raise ValueError("orc_sampled_apply failed")
    return y, tf.value, tr.value


def port_network(current, feed_rows, edge_len, z0):
    """portNetwork restated (postproc.cpp:186-230): dict(y, z, s)."""
    cur = np.asfortranarray(current, dtype=np.complex128)
    p = cur.shape[1]
    feed = np.ascontiguousarray(feed_rows, dtype=np.int64)
    z0 = np.ascontiguousarray(z0, dtype=np.float64)
    out = [np.empty((p, p), np.complex128, order="F") for _ in range(3)]
    st = lib().orc_port_network(_p(cur), cur.shape[0], p, feed.ctypes.data_as(C.POINTER(C.c_longlong)),
                                float(edge_len), z0.ctypes.data_as(dp), *[_p(o) for o in out])
    if st == 1:
        raise ValueError("portNetwork: bad arguments")
    if st == 2:
        raise ArithmeticError("portNetwork: singular admittance matrix")
    return dict(y=out[0], z=out[1], s=out[2])


def array_farfield(nx, ny, e, tensors, dirs, dx, dy, k, eta, current, weights):
    """arrayFarfield restated for the columns of current @ weights: (co, cx)."""
    e = np.ascontiguousarray(e, dtype=np.int32)
    keep = []
    pco, pcx = (dp * 9)(), (dp * 9)()
    for c in range(9):
        if e[c] == 0 or tensors[c] is None:
            pco[c] = pcx[c] = None
            continue
        a = np.asfortranarray(tensors[c][0], dtype=np.complex128)
        b = np.asfortranarray(tensors[c][1], dtype=np.complex128)
        keep += [a, b]
        pco[c], pcx[c] = _p(a), _p(b)
    d = np.ascontiguousarray(dirs, dtype=np.float64)
    cur = np.asfortranarray(current, dtype=np.complex128)
    W = np.asfortranarray(weights, dtype=np.complex128)
    if W.ndim == 1:
        W = W[:, None]
    ndir, q = d.shape[0], W.shape[1]
    co = np.empty((ndir, q), np.complex128, order="F")
    cx = np.empty_like(co)
    lib().orc_array_farfield(nx, ny, e.ctypes.data_as(ip), pco, pcx, ndir, _p(d), dx, dy, k, eta, _p(cur),
                             cur.shape[1], _p(W), q, _p(co), _p(cx))
    return co, cx


# ---------------------------------------------------------------------------
# The reference itself: oracle/_ref/libref_linsolve.so, the reference's own
# linsolve.cpp / toeplitz.cpp / fft.cpp (+ mesh, array_model, partition)
# compiled unchanged against the functional Eigen-subset shim
# (oracle/eigen_shim, oracle/ref_pin/ref_capi.cpp). Pins this oracle.

REF_LINSOLVE_SO = HERE / "_ref" / "libref_linsolve.so"
_refls = None


def ref_linsolve() -> C.CDLL | None:
    """The reference's operator / solver library, or None when not built."""
    global _refls
    if _refls is None and REF_LINSOLVE_SO.exists():
        L = C.CDLL(str(REF_LINSOLVE_SO))
        vp = C.c_void_p
        llp = C.POINTER(C.c_longlong)
        L.refp_last_error.restype = C.c_char_p
        L.refp_load.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.refp_save.argtypes = [vp, C.c_char_p]
        L.refp_destroy.restype = None
        L.refp_destroy.argtypes = [vp]
        L.refp_sizes.argtypes = [vp, llp, llp, ip]
        L.refp_edge_start.argtypes = [vp, llp]
        L.refp_apply.argtypes = [vp, C.c_int, dp, dp]
        L.refp_apply_a_cols.argtypes = [vp, dp, dp, C.c_int, C.c_int]
        L.refp_diagonal.argtypes = [vp, dp]
        L.refp_gmres.argtypes = [vp, dp, dp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, ip, dp, ip, llp]
        L.refp_solve.argtypes = [vp, C.c_int, dp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, dp, ip,
                                 dp]
        L.refp_reconstruct_full.argtypes = [vp, dp]
        L.refp_excitation.argtypes = [vp, C.c_int, ip, C.c_int, llp]
        _refls = L
    return _refls


def write_ztoe1_a(path, nx, ny, m, gen_raw):
    """A-only ZTOE1 block cache (saveBlockCache's format, toeplitz.cpp:
    701-752: "ZTOE1", u8 mode 2 = Sparse, i32 nx, ny, e[9], AGen records
    {u8 1, i32 i, j, 0, i64 rows, cols, column-major complex128}, u8 255)
    from gen.blocks_raw-ordered blocks, for RefOperator."""
    import struct
    e = [0] * 9
    e[4] = m
    g = np.ascontiguousarray(gen_raw, dtype=np.complex128)
    with open(path, "wb") as f:
        f.write(b"ZTOE1" + struct.pack("<Bii9i", 2, nx, ny, *e))
        t = 0
        for i in range(ny):
            for j in range(nx if i == 0 else 2 * nx - 1):
                f.write(struct.pack("<Biiiqq", 1, i, j, 0, m, m))
                f.write(g[t].tobytes())  # raw [t][b][a]: already column-major
                t += 1
        f.write(struct.pack("<B", 255))


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status  # 1 UserError, 2 NumericError, 3 other


class RefOperator:
    """The reference's ToeplitzMatvec over a ZTOE1 block cache (loaded by its
    own loadBlockCache, toeplitz.cpp:754-815), with its own solvers."""

    APPLY, APPLY_A, APPLY_B, APPLY_BT, APPLY_C = range(5)

    def __init__(self, path):
        self._L = ref_linsolve()
        if self._L is None:
            raise ImportError(f"{REF_LINSOLVE_SO} missing: run `make -C oracle ref` where the reference is mounted")
        h = C.c_void_p()
        self._check(self._L.refp_load(str(path).encode(), C.byref(h)))
        self._h = h
        nA, nM, mode = C.c_longlong(), C.c_longlong(), C.c_int()
        self._L.refp_sizes(self._h, C.byref(nA), C.byref(nM), C.byref(mode))
        self.nA, self.nM, self.mode = nA.value, nM.value, mode.value
        self.n = self.nA + self.nM

    def _check(self, st):
        if st:
            raise RefError(st, self._L.refp_last_error().decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.refp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def save(self, path):
        self._check(self._L.refp_save(self._h, str(path).encode()))

    def edge_start(self):
        out = np.zeros(4 * (self.n + 8) + 64, np.int64)
        k = self._L.refp_edge_start(self._h, out.ctypes.data_as(C.POINTER(C.c_longlong)))
        return out[:k].copy()

    def _apply(self, which, x, n_out):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.empty(n_out, np.complex128)
        self._check(self._L.refp_apply(self._h, which, _p(x), _p(y)))
        return y

    def apply(self, x):
        return self._apply(self.APPLY, x, self.n)

    def applyA(self, x):
        return self._apply(self.APPLY_A, x, self.nA)

    def applyB(self, xA):
        return self._apply(self.APPLY_B, xA, self.nM)

    def applyBT(self, xM):
        return self._apply(self.APPLY_BT, xM, self.nA)

    def applyC(self, xM):
        return self._apply(self.APPLY_C, xM, self.nM)

    def apply_a_cols(self, X, threads=1):
        X = np.asfortranarray(X, dtype=np.complex128)
        Y = np.empty_like(X, order="F")
        self._check(self._L.refp_apply_a_cols(self._h, _p(X), _p(Y), X.shape[1], threads))
        return Y

    def diagonal(self):
        d = np.empty(self.n, np.complex128)
        self._check(self._L.refp_diagonal(self._h, _p(d)))
        return d

    def gmres(self, b, tol=1e-8, max_iter=2000, restart=60, precondition=True, use_a_only=False):
        """The reference's own gmres() (linsolve.cpp:425-515) on one column:
        dict(x, iterations, residual, converged, matvecs), partial results
        kept when it does not converge."""
        b = np.ascontiguousarray(b, dtype=np.complex128)
        x = np.empty_like(b)
        it, conv = C.c_int(), C.c_int()
        res = C.c_double()
        mv = C.c_longlong()
        self._check(self._L.refp_gmres(self._h, _p(b), _p(x), 1 if use_a_only else 0, 1 if precondition else 0, tol,
                                       max_iter, restart, C.byref(it), C.byref(res), C.byref(conv), C.byref(mv)))
        return dict(x=x, iterations=it.value, residual=res.value, converged=bool(conv.value), matvecs=mv.value)

    def solve(self, kind, V, tol=1e-8, max_iter=2000, restart=60, precondition=True, threads=1):
        """kind: 'iterative' | 'schur' | 'dense' (linsolve.cpp:532-682).
        Raises RefError(status 1/2) as the reference throws."""
        V = np.asfortranarray(V, dtype=np.complex128)
        vec = V.ndim == 1
        if vec:
            V = V[:, None]
        p = V.shape[1]
        X = np.empty_like(V, order="F")
        its = np.zeros(p, np.int32)
        res = np.zeros(p, np.float64)
        k = {"iterative": 0, "schur": 1, "dense": 2}[kind]
        self._check(self._L.refp_solve(self._h, k, _p(V), p, tol, max_iter, restart, 1 if precondition else 0,
                                       threads, _p(X), its.ctypes.data_as(ip), _p(res)))
        return dict(x=X[:, 0] if vec else X, iterations=its.tolist(), residual=res.tolist())

    def dense(self):
        z = np.empty((self.n, self.n), np.complex128, order="F")
        self._check(self._L.refp_reconstruct_full(self._h, _p(z)))
        return z

    def excitation_rows(self, feed_local_edge, ports):
        pa = np.ascontiguousarray(ports, dtype=np.int32)
        rows = np.zeros(len(pa), np.int64)
        self._check(self._L.refp_excitation(self._h, feed_local_edge, pa.ctypes.data_as(ip), len(pa),
                                            rows.ctypes.data_as(C.POINTER(C.c_longlong))))
        return rows
