"""Parity of the CUDA path (through the C ABI) with the CPU oracle on
identical seeded inputs. Tolerances are the north star's: matvec relative
error <= 1e-11 (complex128); GMRES solution and residual history within
1e-8 relative."""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import (CONFIGS, Config, SolverOptions, ToeplitzMatvec, ToeplitzRep, UserError,
                                   gen, rhs_for)

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-11
GMRES_TOL = 1e-8


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def rep_for(nx, ny, m, seed=1, rank=4, antisym=False, corr=True):
    cfg = Config("t", nx, ny, m, 1, rank, seed, "normal", 20)
    rep = ToeplitzRep.synthetic(cfg)
    if not corr:
        rep.correction = None
    if antisym:
        rng = np.random.default_rng(seed + 99)
        k = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
        rep.generators[0] += 0.3 * (k - k.T)
    return rep


SHAPES = [(4, 4, 24), (1, 1, 5), (1, 5, 3), (6, 1, 4), (3, 5, 7), (5, 3, 8), (7, 9, 64), (9, 5, 128),
          (5, 4, 192), (16, 16, 64), (17, 9, 32)]


@pytest.mark.parametrize("nx,ny,m", SHAPES)
@pytest.mark.parametrize("antisym", [False, True])
def test_apply_matches_oracle(gpu, nx, ny, m, antisym):
    rep = rep_for(nx, ny, m, seed=nx + 7 * ny, antisym=antisym)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    rng = np.random.default_rng(11)
    for _ in range(3):
        x = rng.standard_normal(o.n) + 1j * rng.standard_normal(o.n)
        assert rel(op.apply(x), o.apply(x)) < MATVEC_TOL
        assert rel(op.applyA(x), o.applyA(x)) < MATVEC_TOL
    assert np.array_equal(op.apply(np.zeros(o.n, complex)), np.zeros(o.n, complex))
    assert np.allclose(op.diagonal(), o.diagonal(), rtol=1e-14, atol=0)


SMOOTH_SHAPES = [(18, 9, 8, (36, 18)), (5, 3, 7, (9, 6)), (2, 7, 6, (3, 16)), (10, 12, 12, (24, 24)),
                 (37, 5, 4, (96, 9)), (70, 3, 2, (144, 6)), (90, 2, 3, (192, 3)), (18, 9, 64, (36, 18))]


@pytest.mark.parametrize("nx,ny,m,L", SMOOTH_SHAPES)
def test_smooth_embedding_apply(gpu, nx, ny, m, L):
    """Mixed-radix (2^a 3^b) circulant embedding: a different exact embedding
    of the same operator, so it must agree with the reference's pow2 one."""
    rep = rep_for(nx, ny, m, seed=nx + ny)
    op = ToeplitzMatvec(rep, embed="smooth")
    inf = op.info()
    assert (inf.L0, inf.L1) == L
    o = oracle.Oracle.from_rep(rep)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(o.n) + 1j * rng.standard_normal(o.n)
    assert rel(op.apply(x), o.apply(x)) < MATVEC_TOL
    assert rel(op.applyA(x), o.applyA(x)) < MATVEC_TOL
    op3 = ToeplitzMatvec(rep, embed="smooth", max_nrhs=9)
    X = gen.rhs_normal(o.n, 9, 4)
    Y = op3.apply(X)
    for c in (0, 8):
        assert rel(Y[:, c], o.apply(np.ascontiguousarray(X[:, c]))) < MATVEC_TOL


def test_spectra_bins_match_reference_layout(gpu):
    nx, ny, m = 5, 3, 6
    rep = rep_for(nx, ny, m, antisym=False)
    op = ToeplitzMatvec(rep)
    ah = oracle.Oracle.from_rep(rep).ahat()  # [(m*e5+n)*L + f]
    inf = op.info()
    L0, L1 = 16, 8  # nextPow2(2*5-1), nextPow2(2*3-1)
    assert inf.bins == L0 * L1 and inf.L0 == L0 and inf.L1 == L1
    assert inf.pairs == (L0 * L1 + 4) // 2  # 4 self-paired bins
    for f in range(inf.bins):
        blk = op.spectrum_bin(f)
        assert np.abs(blk - ah[:, :, f]).max() < 1e-13 * np.abs(ah).max(), f


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_apply(gpu, name):
    cfg = CONFIGS[name]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep, nthreads=0)
    x = gen.rhs_normal(cfg.n, 1, 1234)[:, 0]
    assert rel(op.apply(x), o.apply(x)) < MATVEC_TOL
    b = np.asarray(rhs_for(cfg))
    b = b[:, 0] if b.ndim == 2 else b
    assert rel(op.apply(b), o.apply(b)) < MATVEC_TOL


def test_c4_sampled_rows(gpu):
    # Full-size C4 through the direct spatial oracle at sampled elements.
    cfg = CONFIGS["C4"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    x = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
    y = op.apply(x).reshape(cfg.nx * cfg.ny, cfg.m)
    o = oracle.Oracle.from_rep(rep, precompute=False)
    el = [0, 63, 64 * 31 + 17, 64 * 64 - 1]
    yr = o.apply_rows(x, el)
    assert np.linalg.norm(y[el] - yr) / np.linalg.norm(yr) < MATVEC_TOL
    # linearity at full size
    w = gen.rhs_normal(cfg.n, 1, 99)[:, 0]
    a = 0.7 - 0.2j
    assert rel(op.apply(x + a * w), op.apply(x) + a * op.apply(w)) < 1e-13


@pytest.fixture(params=["fused", "passes"])
def fft_path(request, monkeypatch):
    """Both transform paths: cluster-fused 2-D kernels and 1-D line passes."""
    if request.param == "passes":
        monkeypatch.setenv("TBT_FFT", "passes")
    else:
        monkeypatch.delenv("TBT_FFT", raising=False)
    return request.param


@pytest.mark.parametrize("nx,ny,m,k,rank", [(6, 5, 64, 3, 4), (5, 4, 8, 3, 4), (4, 4, 24, 2, 4), (9, 5, 128, 2, 4),
                                            (3, 5, 7, 4, 4), (6, 5, 64, 9, 4), (5, 3, 128, 60, 4), (7, 4, 64, 57, 4),
                                            (6, 5, 64, 33, 8), (5, 3, 128, 40, 8), (4, 6, 128, 8, 8)])
def test_multi_rhs_apply(gpu, fft_path, nx, ny, m, k, rank):
    """k >= 8 with m in {64, 128} and rank 4/8 runs the many-column
    correction kernel (corrMulti), including ragged last 32-column chunks."""
    rep = rep_for(nx, ny, m, rank=rank)
    op = ToeplitzMatvec(rep, max_nrhs=k)
    o = oracle.Oracle.from_rep(rep)
    X = gen.rhs_normal(o.n, k, 5)
    Y = op.apply(X)
    Ya = op.applyA(X)
    for c in range(k):
        xc = np.ascontiguousarray(X[:, c])
        assert rel(Y[:, c], o.apply(xc)) < MATVEC_TOL
        assert rel(Ya[:, c], o.applyA(xc)) < MATVEC_TOL


@pytest.mark.parametrize("orthog", [0, 1])
def test_gmres_single_column_small(gpu, fft_path, orthog):
    rep = rep_for(5, 4, 8, seed=3)
    o = oracle.Oracle.from_rep(rep)
    b = gen.rhs_normal(o.n, 1, 21)[:, 0]
    op = ToeplitzMatvec(rep)
    g = op.gmres(b, SolverOptions(tol=1e-9, maxIter=500, restart=12, orthog=orthog))
    r = o.gmres(b, tol=1e-9, max_iter=500, restart=12)
    assert g.iterations == r["iterations"]
    hist_close(g.history[0], r["history"][0], GMRES_TOL)


@pytest.mark.parametrize("embed", ["pow2", "smooth"])
def test_c3_ports_apply(gpu, embed):
    """C3 (two 9x9 arrays as 18x9, m = 128, 162 unit port columns): the
    bin product is the DMMA batched GEMM; sampled columns vs the oracle.
    The smooth embedding is 36 x 18 bins instead of 64 x 32."""
    cfg = CONFIGS["C3"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep, max_nrhs=cfg.nrhs, embed=embed)
    V = np.asarray(rhs_for(cfg))
    assert V.shape == (cfg.n, 162)
    Y = op.apply(V)
    o = oracle.Oracle.from_rep(rep, nthreads=0)
    for c in [0, 17, 80, 161]:
        assert rel(Y[:, c], o.apply(np.ascontiguousarray(V[:, c]))) < MATVEC_TOL
    # linearity across columns: Z (V a) = (Z V) a
    a = gen.rhs_normal(162, 1, 5)[:, 0]
    assert rel(op.apply(V @ a), Y @ a) < 1e-12


def test_c5_full_size_sampled(gpu):
    """C5 (128x128, m = 192; 19.2 GB of generator blocks, 19.3 GB stored half
    spectrum): full-size apply checked at sampled elements against the
    direct spatial sum (no FFT), plus linearity."""
    import psutil
    if psutil.virtual_memory().total < 70 * 2**30:
        pytest.skip("needs >= 70 GB host memory for the C5 generators + oracle copy")
    cfg = CONFIGS["C5"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    x = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
    y = op.apply(x).reshape(cfg.nx * cfg.ny, cfg.m)
    o = oracle.Oracle.from_rep(rep, precompute=False)
    rep.generators = None  # drop the numpy copy; the oracle holds its own
    el = [0, 127 * 128 + 5, 64 * 128 + 64]
    yr = o.apply_rows(x, el)
    o.close()
    assert np.linalg.norm(y[el] - yr) / np.linalg.norm(yr) < MATVEC_TOL
    w = gen.rhs_normal(cfg.n, 1, 98)[:, 0]
    assert rel(op.apply(x - 0.5j * w), op.apply(x) - 0.5j * op.apply(w)) < 1e-13


def test_user_errors(gpu):
    op = ToeplitzMatvec(rep_for(3, 3, 4))
    with pytest.raises(UserError):
        op.apply(np.zeros(5, complex))
    with pytest.raises(UserError):
        ToeplitzMatvec(ToeplitzRep(3, 3, 4, np.zeros((3, 4, 4), complex)))


HIST_ATOL = 1e-14  # residuals are normalised (first entry 1): the double-precision floor


def hist_close(h_gpu, h_ref, tol):
    """Same event sequence (restart / inner / final), values within
    |d| <= tol*|h| + 1e-14. History values are residuals relative to ||b||
    or beta, so 1e-14 is the rounding floor two correct complex128 GMRES
    implementations share (reduction order differs); near convergence
    (h ~ 1e-9) a pure relative 1e-8 test would sit below that floor."""
    assert h_gpu.shape == h_ref.shape, (h_gpu.shape, h_ref.shape)
    assert np.array_equal(h_gpu[:, 0], h_ref[:, 0])
    d = np.abs(h_gpu[:, 1] - h_ref[:, 1])
    bound = tol * np.abs(h_ref[:, 1]) + HIST_ATOL
    assert np.all(d <= bound), (d / bound).max()


@pytest.mark.parametrize("orthog", [0, 1])
def test_gmres_c1_parity(gpu, orthog):
    cfg = CONFIGS["C1"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    b = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
    opt = SolverOptions(tol=cfg.tol, maxIter=cfg.max_iter, restart=cfg.restart, orthog=orthog)
    g = op.gmres(b, opt)
    r = o.gmres(b, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart)
    assert g.converged == [1] and r["converged"] == [1]
    assert g.iterations == r["iterations"]
    assert rel(g.current, r["x"]) < GMRES_TOL
    hist_close(g.history[0], r["history"][0], GMRES_TOL)


@pytest.mark.parametrize("orthog", [0, 1])
def test_gmres_c2_budget_parity(gpu, orthog):
    # C2 stalls under GMRES(50)+Jacobi: compare a fixed
    # 200-iteration budget (4 restarts, the bench's budget) history and iterate.
    cfg = CONFIGS["C2"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    b = rhs_for(cfg)
    opt = SolverOptions(tol=cfg.tol, maxIter=200, restart=cfg.restart, orthog=orthog)
    g = op.gmres(b, opt, raise_on_fail=False)
    r = o.gmres(b, tol=cfg.tol, max_iter=200, restart=cfg.restart)
    assert g.iterations == r["iterations"] == [200]
    hist_close(g.history[0], r["history"][0], GMRES_TOL)
    assert rel(g.current, r["x"]) < GMRES_TOL


@pytest.mark.parametrize("orthog", [0, 1])
def test_gmres_multi_column_and_a_only(gpu, fft_path, orthog):
    """Columns in lockstep; orthog=1 runs the batched low-sync Arnoldi
    (lsCols* kernels), orthog=0 the per-column MGS sweep."""
    rep = rep_for(5, 4, 8, seed=3)
    o = oracle.Oracle.from_rep(rep)
    B = gen.rhs_normal(o.n, 3, 21)
    B[:, 1] = 0.0  # zero column converges immediately (bnorm == 0)
    op = ToeplitzMatvec(rep, max_nrhs=3)
    for a_only in (False, True):
        opt = SolverOptions(tol=1e-9, maxIter=500, restart=12, orthog=orthog)
        g = op.gmres(B, opt, use_a_only=a_only)
        r = o.gmres(B, tol=1e-9, max_iter=500, restart=12, use_a_only=a_only)
        assert g.iterations == r["iterations"]
        assert g.converged == r["converged"] == [1, 1, 1]
        for c in range(3):
            if c == 1:
                assert not np.any(g.current[:, c])
                continue
            assert rel(g.current[:, c], r["x"][:, c]) < GMRES_TOL
            hist_close(g.history[c], r["history"][c], GMRES_TOL)


@pytest.mark.parametrize("nx,ny,m,k,orthog", [(4, 3, 128, 10, 1), (6, 5, 64, 20, 1), (4, 3, 128, 10, 0),
                                              (3, 3, 200, 5, 1)])
def test_gmres_many_columns(gpu, nx, ny, m, k, orthog):
    """Many columns at C3-like basis sizes (one warp per element, m/32 values
    per lane); columns stop at different iterations and restarts."""
    rep = rep_for(nx, ny, m, seed=5, rank=8)
    o = oracle.Oracle.from_rep(rep)
    B = gen.rhs_normal(o.n, k, 33)
    B[:, 1] *= 1e-3
    op = ToeplitzMatvec(rep, max_nrhs=k)
    opt = SolverOptions(tol=1e-8, maxIter=300, restart=15, orthog=orthog)
    g = op.gmres(B, opt, raise_on_fail=False)
    r = o.gmres(B, tol=1e-8, max_iter=300, restart=15)
    assert g.iterations == r["iterations"]
    assert g.converged == r["converged"]
    for c in range(k):
        assert rel(g.current[:, c], r["x"][:, c]) < GMRES_TOL
        hist_close(g.history[c], r["history"][c], GMRES_TOL)


def test_gmres_nonconvergence_raises(gpu):
    from paper_2506_04710_b200 import NumericError
    rep = rep_for(4, 4, 8)
    op = ToeplitzMatvec(rep)
    b = gen.rhs_normal(op.sizeA(), 1, 3)[:, 0]
    with pytest.raises(NumericError):
        op.gmres(b, SolverOptions(tol=1e-15, maxIter=7, restart=3))


@pytest.mark.gpu
@pytest.mark.parametrize("corr", [True, False])
def test_zero_copy_pinned_apply(gpu, corr):
    """Pinned host x / y take the zero-copy persistent launch (x read over
    PCIe in phase A1 and staged for the correction terms, spectrum
    L2-prefetched meanwhile): identical to the device-resident apply."""
    import ctypes as C

    import torch

    from paper_2506_04710_b200._lib import TBT_DEVICE, TBT_HOST, lib
    cfg = CONFIGS["C2"]
    rep = ToeplitzRep.synthetic(cfg)
    if not corr:
        rep.correction = None
    op = ToeplitzMatvec(rep)
    x = gen.rhs_normal(cfg.n, 1, 17)[:, 0]
    xh = torch.from_numpy(x.copy()).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    xd, yd = xh.cuda(), torch.empty(cfg.n, dtype=torch.complex128, device="cuda")
    for _ in range(3):  # repeated calls replay the cached zero-copy graph
        assert lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST) == 0
    assert lib().tbt_apply(op._h, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), 1, TBT_DEVICE) == 0
    torch.cuda.synchronize()
    assert np.array_equal(yh.numpy(), yd.cpu().numpy())
    o = oracle.Oracle.from_rep(rep, nthreads=0)
    ref = o.apply(x)
    assert rel(yh.numpy(), ref) < MATVEC_TOL


@pytest.mark.gpu
def test_concurrent_callers_one_context(gpu):
    """The reference calls apply from parallelFor workers (linsolve.cpp:572);
    concurrent callers on one context are serialised by the context lock and
    every result matches a serial apply."""
    import threading
    rep = ToeplitzRep.synthetic(Config("thr", 6, 5, 8, 1, 2, 21, "normal", 20))
    op = ToeplitzMatvec(rep)
    xs = [gen.rhs_normal(op.size(), 1, 40 + t)[:, 0] for t in range(4)]
    ref = [op.apply(x) for x in xs]
    errors = []

    def worker(t):
        try:
            for _ in range(25):
                if not np.array_equal(op.apply(xs[t]), ref[t]):
                    errors.append(t)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors


# Persistent single-kernel apply instantiated beyond the BASELINE shapes
# (matvec_persistent.cu): (m, L0, L1) -> a grid that selects it.
PERSISTENT_EXTRA = [(33, 33, 96), (40, 24, 64), (24, 40, 64), (40, 40, 64), (20, 17, 128), (65, 70, 128), (40, 36, 192)]


@pytest.mark.parametrize("nx,ny,m", PERSISTENT_EXTRA)
def test_persistent_extra_shapes(gpu, nx, ny, m):
    rep = ToeplitzRep.synthetic(Config("pe", nx, ny, m, 1, 8, 4, "normal", 50))
    op = ToeplitzMatvec(rep)
    assert op.info().apply_path == 2, "expected the persistent kernel"
    x = gen.rhs_normal(nx * ny * m, 1, 3)[:, 0]
    y = op.apply(x).reshape(nx * ny, m)
    o = oracle.Oracle.from_rep(rep, precompute=False)
    el = [0, nx - 1, (ny // 2) * nx + nx // 3, nx * ny - nx, nx * ny - 1]
    yr = o.apply_rows(x, el)
    assert np.linalg.norm(y[el] - yr) / np.linalg.norm(yr) < MATVEC_TOL
    # single-column GMRES through the persistent kernel (fused LS step where
    # the row chunk fits shared memory, the streamed one otherwise)
    g = op.gmres(x, SolverOptions(tol=1e-8, maxIter=12, restart=10), raise_on_fail=False)
    assert g.iterations[0] == 12 and np.isfinite(g.residual[0])
    if nx * ny * m <= 70000:  # the oracle's spectra are cheap here: full GMRES parity
        o.precompute()
        r = o.gmres(x, tol=1e-8, max_iter=12, restart=10)
        assert g.iterations == r["iterations"] and rel(g.current, r["x"]) < 1e-8
        h, hr = g.history[0], r["history"][0]
        assert h.shape == hr.shape and np.all(np.abs(h[:, 1] - hr[:, 1]) <= 1e-8 * np.abs(hr[:, 1]) + 1e-14)
