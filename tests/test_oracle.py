"""The CPU oracle, pinned before it is trusted.

* fftInPlace (proj/src/fft.cpp:28-53) is pinned BITWISE against the
  reference's own fft.cpp: live through oracle/_ref when it was built, and
  through tests/golden/ref_fft.npz (made from oracle/_ref by
  tests/golden/make_golden.py) everywhere.
* The restated applyA / gmres have no reference golden vectors (the
  reference's tests/ are not mounted and Eigen is absent, so the reference
  matvec cannot run): they are pinned on SPEC.md's known-answer properties
   against an independent dense numpy
  product / LU solve.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import CONFIGS, Config, ToeplitzRep, gen

GOLD = Path(__file__).resolve().parent / "golden" / "ref_fft.npz"


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_fft_bitwise_vs_reference_golden():
    g = np.load(GOLD)
    for n in [1, 2, 4, 8, 16, 32, 64, 128, 256]:
        x = g[f"in_{n}"]
        assert np.array_equal(bits(oracle.fft(x)), bits(g[f"fwd_{n}"])), n
        assert np.array_equal(bits(oracle.fft(x, inverse=True)), bits(g[f"inv_{n}"])), n
    for k, v in g["next_pow2"]:
        assert oracle.lib().orc_next_pow2(int(k)) == v


@pytest.mark.skipif(oracle.ref_lib() is None, reason="oracle/_ref not built")
def test_fft_bitwise_vs_reference_live():
    rng = np.random.default_rng(1)
    for n in [2, 8, 64, 512, 2048]:
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        for inv in (False, True):
            assert np.array_equal(bits(oracle.fft(x, inv)), bits(oracle.ref_fft(x, inv)))
    with pytest.raises(ValueError):
        oracle.ref_fft(np.ones(6, complex))


def test_fft_semantics():
    rng = np.random.default_rng(2)
    x = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    assert np.allclose(oracle.fft(x), np.fft.fft(x), rtol=0, atol=1e-12)
    # unscaled inverse (fft.hpp:27-28)
    assert np.allclose(oracle.fft(x, True), np.fft.ifft(x) * 64, rtol=0, atol=1e-12)
    with pytest.raises(ValueError):
        oracle.fft(np.ones(12, complex))


def small_rep(nx, ny, m, seed=0, rank=4, antisym=False):
    cfg = Config("t", nx, ny, m, 1, rank, seed, "normal", 20)
    rep = ToeplitzRep.synthetic(cfg)
    if antisym:
        rng = np.random.default_rng(seed + 99)
        k = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
        rep.generators[0] += 0.3 * (k - k.T)
    return rep


SHAPES = [(4, 4, 24), (1, 1, 5), (1, 5, 3), (6, 1, 4), (3, 5, 7), (5, 3, 8), (2, 7, 6)]


@pytest.mark.parametrize("nx,ny,m", SHAPES)
@pytest.mark.parametrize("antisym", [False, True])
def test_matvec_vs_dense(nx, ny, m, antisym):
    rep = small_rep(nx, ny, m, seed=nx * 10 + ny, antisym=antisym)
    o = oracle.Oracle.from_rep(rep)
    Z = o.dense()
    rng = np.random.default_rng(5)
    for _ in range(5):
        x = rng.standard_normal(o.n) + 1j * rng.standard_normal(o.n)
        yd = Z @ x
        assert np.linalg.norm(o.apply(x) - yd) / np.linalg.norm(yd) < 1e-12
    # applyA alone = Toeplitz part: dense without correction
    o2 = oracle.Oracle.from_rep(ToeplitzRep(rep.nx, rep.ny, rep.m, rep.generators, None))
    Za = o2.dense()
    assert np.linalg.norm(o.applyA(x) - Za @ x) / np.linalg.norm(Za @ x) < 1e-12
    # rows oracle (direct spatial sum) agrees with dense
    el = [0, nx * ny - 1, (nx * ny) // 2]
    yr = o.apply_rows(x, el)
    assert np.abs(yr - yd.reshape(nx * ny, m)[el]).max() / np.abs(yd).max() < 1e-13


def test_matvec_zero_and_linearity():
    o = oracle.Oracle.from_rep(small_rep(4, 4, 24))
    assert not np.any(o.apply(np.zeros(o.n, complex)))
    rng = np.random.default_rng(3)
    x = rng.standard_normal(o.n) + 1j * rng.standard_normal(o.n)
    w = rng.standard_normal(o.n) + 1j * rng.standard_normal(o.n)
    a, b = 0.3 - 1.2j, 2.0 + 0.5j
    lhs = o.apply(a * x + b * w)
    rhs = a * o.apply(x) + b * o.apply(w)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-12


def test_reciprocal_generator_gives_symmetric_operator():
    o = oracle.Oracle.from_rep(small_rep(4, 3, 6))
    Z = o.dense()
    assert np.abs(Z - Z.T).max() < 1e-14 * np.abs(Z).max()


def test_embedding_roundtrip():
    # embedding then extracting the generator sequence is the
    # identity: inverse 2-D DFT of ahat returns aEntry at every shift.
    nx, ny, m = 3, 4, 5
    rep = small_rep(nx, ny, m, antisym=True)
    o = oracle.Oracle.from_rep(rep)
    ah = o.ahat()
    L1, L0 = 8, 8
    grid = np.fft.ifft2(ah.reshape(m, m, L1, L0), axes=(2, 3))
    raw = rep.generators  # [t][b][a]
    for t in range(gen.num_blocks(nx, ny)):
        i, j = gen.block_shift(nx, ny, t)
        blk = raw[t].T  # [a][b]
        assert np.allclose(grid[:, :, i % L1, j % L0], blk, atol=1e-14)
        if (i, j) != (0, 0):
            assert np.allclose(grid[:, :, (-i) % L1, (-j) % L0], blk.T, atol=1e-14)


def test_diagonal():
    o = oracle.Oracle.from_rep(small_rep(5, 3, 8))
    assert np.allclose(o.diagonal(), np.diag(o.dense()), rtol=0, atol=1e-14)


def test_gmres_c1_vs_dense():
    cfg = CONFIGS["C1"]
    rep = ToeplitzRep.synthetic(cfg)
    o = oracle.Oracle.from_rep(rep)
    Z = o.dense()
    b = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
    r = o.gmres(b, tol=1e-10, restart=cfg.restart)
    assert r["converged"] == [1]
    xs = np.linalg.solve(Z, b)
    assert np.linalg.norm(r["x"] - xs) / np.linalg.norm(xs) < 1e-8
    h = r["history"][0]
    assert h[0, 0] == 0 and h[0, 1] == pytest.approx(1.0)  # x0 = 0 -> first residual 1
    assert np.all(np.diff(h[h[:, 0] == 1][:, 1][: cfg.restart]) <= 1e-15)  # monotone in a cycle


def test_gmres_recovers_unit_vector():
    o = oracle.Oracle.from_rep(small_rep(3, 3, 6))
    e1 = np.zeros(o.n, complex)
    e1[0] = 1
    v = o.apply(e1)  # V = Z e1 recovers e1
    r = o.gmres(v, tol=1e-10, restart=30)
    assert r["converged"] == [1]
    assert np.linalg.norm(r["x"] - e1) < 1e-8


def test_gmres_jacobi_not_worse():
    o = oracle.Oracle.from_rep(small_rep(4, 4, 8, seed=3))
    b = gen.rhs_normal(o.n, 1, 11)[:, 0]
    r1 = o.gmres(b, tol=1e-8, restart=30, precondition=True)
    r0 = o.gmres(b, tol=1e-8, restart=30, precondition=False)
    assert r1["converged"] == [1] and r0["converged"] == [1]
    assert r1["iterations"][0] <= r0["iterations"][0]


def test_gmres_max_iter_reports_partial():
    o = oracle.Oracle.from_rep(small_rep(4, 4, 8))
    b = gen.rhs_normal(o.n, 1, 4)[:, 0]
    r = o.gmres(b, tol=1e-14, restart=5, max_iter=12)
    assert r["converged"] == [0] and r["iterations"] == [12]
    kinds = r["history"][0][:, 0]
    assert list(kinds).count(1.0) == 12 and kinds[-1] == 2.0


def test_gmres_multi_column_threads_match_serial():
    o = oracle.Oracle.from_rep(small_rep(3, 3, 6))
    B = gen.rhs_normal(o.n, 4, 8)
    a = o.gmres(B, tol=1e-9, restart=10, nthreads=1)
    b = o.gmres(B, tol=1e-9, restart=10, nthreads=4)
    assert np.array_equal(a["x"], b["x"])  # per-slot writes: schedule independent (common.hpp:52-54)
