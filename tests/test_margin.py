"""Margin coupling B / B^T / C (reference
ToeplitzMatvec::apply with margin parts, proj/src/linsolve.cpp:54-134,
179-216, 292-349, 373-388).

CPU: the oracle's Toe1D restatement against an independent dense assembly of
Z = [A + P, B^T; B, C] from the generator definitions (include/tbt_gen.h),
and GMRES on it against a dense LU solve. GPU: apply / diagonal / GMRES of
the CUDA path against the oracle through the C ABI."""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import Config, SolverOptions, ToeplitzRep, gen

# (nx, ny, m, e[9]) -- e[4] == m; zeros exercise empty components.
SHAPES = [
    (4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]),
    (5, 4, 8, [0, 2, 0, 3, 8, 1, 0, 2, 1]),
    (3, 5, 4, [1, 0, 2, 0, 4, 0, 1, 3, 0]),
    (1, 3, 5, [1, 2, 1, 2, 5, 2, 1, 2, 1]),
    (6, 1, 3, [0, 0, 0, 0, 3, 0, 0, 0, 0]),
]


def rep_with_margin(nx, ny, m, e, seed=3, corr=True):
    rep = ToeplitzRep.synthetic(Config("mg", nx, ny, m, 1, 2 if corr else -1, seed, "normal", 20,
                                       scale=0.1 if corr else 0.0))
    rep.margin = gen.margin(nx, ny, e, seed + 100)
    return rep


def dense_full(rep):
    """Z = [A (+correction), B^T; B, C] assembled entry by entry."""
    nx, ny, m, mg = rep.nx, rep.ny, rep.m, rep.margin
    e = mg.e
    o = oracle.Oracle.from_rep(ToeplitzRep(nx, ny, m, rep.generators, rep.correction), precompute=False)
    A = o.dense()
    nA, nM = nx * ny * m, mg.size(nx, ny)
    B = np.zeros((nM, nA), complex)
    side_start = [0, ny * e[1]]
    row_start = [ny * (e[1] + e[7]), ny * (e[1] + e[7]) + nx * e[5]]
    off = 0
    for r, comp in enumerate((2, 8)):
        em = e[comp - 1]
        blocks = mg.bside[off:off + (2 * ny - 1) * em * nx * m].reshape(2 * ny - 1, nx * m, em)  # col-major
        off += (2 * ny - 1) * em * nx * m
        for a in range(ny):
            for b in range(ny):
                G = blocks[(a - b) + ny - 1].T  # em x nx*m
                B[side_start[r] + a * em: side_start[r] + (a + 1) * em, b * nx * m:(b + 1) * nx * m] = G
    off = 0
    for r, comp in enumerate((6, 4)):
        em = e[comp - 1]
        blocks = mg.brow[off:off + ny * (2 * nx - 1) * em * m].reshape(ny, 2 * nx - 1, m, em)
        off += ny * (2 * nx - 1) * em * m
        for j in range(ny):
            for a in range(nx):
                for b in range(nx):
                    G = blocks[j, (a - b) + nx - 1].T  # em x m
                    B[row_start[r] + a * em: row_start[r] + (a + 1) * em, (j * nx + b) * m:(j * nx + b + 1) * m] = G
    cs = row_start[1] + nx * e[3]
    off = 0
    for comp in (3, 9, 1, 7):
        em = e[comp - 1]
        B[cs:cs + em, :] = mg.bcorner[off:off + em * nA].reshape(nA, em).T
        off += em * nA
        cs += em
    C = mg.c.reshape(nM, nM).T
    return np.block([[A, B.T], [B, C]])


@pytest.mark.parametrize("nx,ny,m,e", SHAPES)
def test_oracle_margin_matches_dense(nx, ny, m, e):
    rep = rep_with_margin(nx, ny, m, e)
    o = oracle.Oracle.from_rep(rep)
    Z = dense_full(rep)
    assert o.n == Z.shape[0] == nx * ny * m + rep.margin.size(nx, ny)
    X = gen.rhs_normal(o.n, 3, 7)
    for c in range(3):
        x = np.ascontiguousarray(X[:, c])
        y = o.apply(x)
        assert np.linalg.norm(y - Z @ x) / np.linalg.norm(Z @ x) < 1e-13
    assert np.allclose(o.diagonal(), np.diag(Z), rtol=0, atol=1e-14)
    # symmetric (reciprocal) when the correction is off: Z = Z^T
    rep0 = rep_with_margin(nx, ny, m, e, corr=False)
    Z0 = dense_full(rep0)
    assert np.linalg.norm(Z0 - Z0.T) < 1e-12 * np.linalg.norm(Z0)


def test_oracle_margin_gmres_vs_lu():
    rep = rep_with_margin(4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1])
    o = oracle.Oracle.from_rep(rep)
    Z = dense_full(rep)
    b = gen.rhs_normal(o.n, 1, 9)[:, 0]
    r = o.gmres(b, tol=1e-10, max_iter=2000, restart=40)
    assert r["converged"] == [1]
    xs = np.linalg.solve(Z, b)
    assert np.linalg.norm(r["x"] - xs) / np.linalg.norm(xs) < 1e-8


def test_margin_generator_layout():
    nx, ny, m, e = 4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]
    mg = gen.margin(nx, ny, e, 5)
    assert mg.bside.size == (2 * ny - 1) * (e[1] + e[7]) * nx * m
    assert mg.brow.size == ny * (2 * nx - 1) * (e[5] + e[3]) * m
    assert mg.bcorner.size == (e[2] + e[8] + e[0] + e[6]) * nx * ny * m
    nM = mg.size(nx, ny)
    C = mg.c.reshape(nM, nM)
    assert np.array_equal(C, C.T)
    assert np.allclose(np.diag(C).real, 2.0, atol=0.5) and np.allclose(np.diag(C).imag, 2.0, atol=0.5)
    mg2 = gen.margin(nx, ny, e, 5)
    assert np.array_equal(mg.bside, mg2.bside) and np.array_equal(mg.c, mg2.c)


@pytest.mark.gpu
# The last two shapes take the wide single-column kernels (9..16 rows per
# margin part) and two corner passes (> 16 corner rows).
@pytest.mark.parametrize("nx,ny,m,e", SHAPES + [(8, 6, 64, [3, 5, 2, 4, 64, 6, 1, 7, 2]),
                                               (4, 3, 6, [5, 12, 6, 10, 6, 9, 5, 11, 4]),
                                               (3, 7, 5, [9, 16, 1, 3, 5, 14, 8, 2, 0])])
@pytest.mark.parametrize("k", [1, 3])
def test_gpu_margin_apply(gpu, nx, ny, m, e, k):
    from paper_2506_04710_b200 import ToeplitzMatvec
    rep = rep_with_margin(nx, ny, m, e)
    op = ToeplitzMatvec(rep, max_nrhs=k)
    o = oracle.Oracle.from_rep(rep)
    assert op.sizeM() == rep.margin.size(nx, ny) and op.size() == o.n
    X = gen.rhs_normal(o.n, k, 11)
    Y = op.apply(X if k > 1 else X[:, 0]).reshape(o.n, k)
    for c in range(k):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert np.linalg.norm(Y[:, c] - ref) / np.linalg.norm(ref) < 1e-11
    # applyA ignores the margin
    ya = op.applyA(np.ascontiguousarray(X[:o.nA, 0]))
    assert np.linalg.norm(ya - o.applyA(np.ascontiguousarray(X[:o.nA, 0]))) < 1e-11 * np.linalg.norm(ya)
    assert np.allclose(op.diagonal(), o.diagonal(), rtol=1e-14, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,m,e", SHAPES[:4] + [(4, 3, 6, [5, 12, 6, 10, 6, 9, 5, 11, 4])])
@pytest.mark.parametrize("k", [1, 2])
def test_gpu_margin_blocks(gpu, nx, ny, m, e, k):
    """applyB / applyBT / applyC (linsolve.hpp:66-68) against the oracle's
    full operator on [xA; 0] and [0; xM]."""
    from paper_2506_04710_b200 import ToeplitzMatvec
    rep = rep_with_margin(nx, ny, m, e)
    op = ToeplitzMatvec(rep, max_nrhs=k)
    o = oracle.Oracle.from_rep(rep)
    nA, nM = op.sizeA(), op.sizeM()
    X = gen.rhs_normal(nA + nM, k, 17)
    for c in range(k):
        xa = np.concatenate([X[:nA, c], np.zeros(nM, complex)])
        xm = np.concatenate([np.zeros(nA, complex), X[nA:, c]])
        ya, ym = o.apply(xa), o.apply(xm)
        got_b = op.applyB(X[:nA, c:c + 1])[:, 0] if k > 1 else op.applyB(X[:nA, c])
        got_bt = op.applyBT(X[nA:, c:c + 1])[:, 0] if k > 1 else op.applyBT(X[nA:, c])
        got_c = op.applyC(X[nA:, c:c + 1])[:, 0] if k > 1 else op.applyC(X[nA:, c])
        for got, ref in ((got_b, ya[nA:]), (got_bt, ym[:nA]), (got_c, ym[nA:])):
            assert np.linalg.norm(got - ref) <= 1e-11 * max(np.linalg.norm(ref), 1e-300)
    Yb = op.applyB(X[:nA])  # all columns at once
    assert Yb.shape == (nM, k)


@pytest.mark.gpu
def test_gpu_margin_blocks_need_margin(gpu):
    from paper_2506_04710_b200 import ToeplitzMatvec, UserError
    rep = rep_with_margin(4, 3, 6, SHAPES[0][3])
    rep.margin = None
    op = ToeplitzMatvec(rep)
    with pytest.raises(UserError):
        op.applyB(np.zeros(op.sizeA(), complex))


@pytest.mark.gpu
@pytest.mark.parametrize("k,orthog", [(1, 1), (3, 1), (2, 0)])
def test_gpu_margin_gmres(gpu, k, orthog):
    from paper_2506_04710_b200 import ToeplitzMatvec
    rep = rep_with_margin(5, 4, 8, [2, 3, 1, 4, 8, 2, 3, 5, 1])
    op = ToeplitzMatvec(rep, max_nrhs=k)
    o = oracle.Oracle.from_rep(rep)
    B = gen.rhs_normal(o.n, k, 13)
    g = op.gmres(B if k > 1 else B[:, 0], SolverOptions(tol=1e-9, maxIter=400, restart=20, orthog=orthog),
                 raise_on_fail=False)
    r = o.gmres(B if k > 1 else B[:, 0], tol=1e-9, max_iter=400, restart=20)
    assert g.iterations == r["iterations"] and g.converged == r["converged"]
    G = np.asarray(g.current).reshape(o.n, k)
    R = np.asarray(r["x"]).reshape(o.n, k)
    for c in range(k):
        assert np.linalg.norm(G[:, c] - R[:, c]) / np.linalg.norm(R[:, c]) < 1e-8
        h, hr = g.history[c], r["history"][c]
        assert h.shape == hr.shape and np.array_equal(h[:, 0], hr[:, 0])
        assert np.all(np.abs(h[:, 1] - hr[:, 1]) <= 1e-8 * np.abs(hr[:, 1]) + 1e-14)
    # A-only solves stay on the element unknowns (schurSolve's inner solves)
    ga = op.gmres(np.ascontiguousarray(B[:o.nA, 0]), SolverOptions(tol=1e-9, maxIter=400, restart=20),
                  use_a_only=True, raise_on_fail=False)
    ra = o.gmres(np.ascontiguousarray(B[:o.nA, 0]), tol=1e-9, max_iter=400, restart=20, use_a_only=True)
    assert ga.iterations == ra["iterations"]
    assert np.linalg.norm(ga.current - ra["x"]) / np.linalg.norm(ra["x"]) < 1e-8


def test_oracle_schur_vs_dense():
    """schurSolve restated (linsolve.cpp:595-682) equals the dense solve of
    Z x = [v; 0], and rejects excitations on margin rows."""
    rep = rep_with_margin(4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1], corr=False)
    o = oracle.Oracle.from_rep(rep)
    Z = dense_full(rep)
    V = np.zeros((o.n, 2), complex)
    V[:o.nA] = gen.rhs_normal(o.nA, 2, 4)
    r = o.schur(V, tol=1e-12, max_iter=3000, restart=40)
    xs = np.linalg.solve(Z, V)
    assert np.linalg.norm(r["x"] - xs) / np.linalg.norm(xs) < 1e-9
    assert max(r["residual"]) < 1e-9
    bad = V.copy()
    bad[-1, 0] = 1.0
    with pytest.raises(ValueError):
        o.schur(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,m,e,p,maxrhs", [(4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1], 2, 8),
                                                 (5, 4, 8, [0, 2, 0, 3, 8, 1, 0, 2, 1], 1, 16),
                                                 (3, 3, 4, [1, 1, 1, 1, 4, 1, 1, 1, 1], 3, 4)])
def test_gpu_schur_solve(gpu, nx, ny, m, e, p, maxrhs):
    """schurSolve on the device (row f2) against the oracle's restatement
    and the dense solve: inner iterations, solution, residual."""
    from paper_2506_04710_b200 import ToeplitzMatvec
    rep = rep_with_margin(nx, ny, m, e, corr=False)
    o = oracle.Oracle.from_rep(rep)
    op = ToeplitzMatvec(rep, max_nrhs=maxrhs)
    V = np.zeros((o.n, p), complex)
    V[:o.nA] = gen.rhs_normal(o.nA, p, 4)
    opt = SolverOptions(tol=1e-11, maxIter=3000, restart=30)
    g = op.schur_solve(V, opt)
    r = o.schur(V, tol=1e-11, max_iter=3000, restart=30)
    assert g.iterations == r["iterations"]
    assert np.linalg.norm(g.current - r["x"]) / np.linalg.norm(r["x"]) < 1e-8
    xs = np.linalg.solve(dense_full(rep), V)
    assert np.linalg.norm(g.current - xs) / np.linalg.norm(xs) < 1e-8
    assert max(g.residual) < 1e-8


@pytest.mark.gpu
def test_gpu_schur_errors(gpu):
    from paper_2506_04710_b200 import NumericError, ToeplitzMatvec, UserError
    rep = rep_with_margin(4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1], corr=False)
    op = ToeplitzMatvec(rep, max_nrhs=4)
    V = np.zeros((op.size(), 1), complex)
    V[:op.sizeA(), 0] = gen.rhs_normal(op.sizeA(), 1, 4)[:, 0]
    bad = V.copy()
    bad[-1, 0] = 1.0
    with pytest.raises(UserError):
        op.schur_solve(bad, SolverOptions())
    with pytest.raises(NumericError):  # inner solves cannot converge in 2 iterations
        op.schur_solve(V, SolverOptions(tol=1e-14, maxIter=2, restart=2))
