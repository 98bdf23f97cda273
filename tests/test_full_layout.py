"""FULL generator layout: every shift's block, for
non-reciprocal operators that the reference's Sparse ToeplitzRep cannot hold
(toeplitz.hpp:72-74). tbt_set_generators_full splits the input into a
reciprocal part (the usual half spectrum) and an anti-reciprocal part
(A_a(-s) = -A_a(s)^T, a second half spectrum whose partner product is
negated). CPU: the oracle's FULL restatement against a dense numpy assembly
and against its Sparse mode on reciprocal input. GPU: apply (1 and 3
columns, several m, with the edge/corner correction), diagonal and GMRES
against the oracle."""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import Config, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen


def full_blocks(nx, ny, m, seed, reciprocal=False):
    """(2ny-1)(2nx-1) raw blocks ([t][b][a] column-major), t = (i+ny-1)*(2nx-1) + (j+nx-1)."""
    rng = np.random.default_rng(seed)
    nb = (2 * ny - 1) * (2 * nx - 1)
    z = (rng.standard_normal((nb, m, m)) + 1j * rng.standard_normal((nb, m, m))) / np.sqrt(m)
    z[(ny - 1) * (2 * nx - 1) + nx - 1] += (3 + 3j) * np.eye(m)  # self block, diagonally dominant-ish
    if reciprocal:  # Z(-s) = Z(s)^T
        for i in range(1 - ny, ny):
            for j in range(1 - nx, nx):
                if i < 0 or (i == 0 and j < 0):
                    t = (i + ny - 1) * (2 * nx - 1) + (j + nx - 1)
                    u = (-i + ny - 1) * (2 * nx - 1) + (-j + nx - 1)
                    z[t] = z[u].T
    return np.ascontiguousarray(z)


def sparse_from_full(nx, ny, full):
    out = []
    for i in range(ny):
        for j in range(0 if i == 0 else 1 - nx, nx):
            out.append(full[(i + ny - 1) * (2 * nx - 1) + (j + nx - 1)])
    return np.ascontiguousarray(np.stack(out))


def dense(nx, ny, m, full):
    n = nx * ny * m
    Z = np.zeros((n, n), complex)
    for rt in range(ny):
        for ct in range(nx):
            for rs in range(ny):
                for cs in range(nx):
                    t = (rt - rs + ny - 1) * (2 * nx - 1) + (ct - cs + nx - 1)
                    et, es = rt * nx + ct, rs * nx + cs
                    Z[et * m:(et + 1) * m, es * m:(es + 1) * m] = full[t].T  # raw [b][a] -> (a, b)
    return Z


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("nx,ny,m", [(3, 2, 4), (1, 4, 3), (4, 1, 2), (3, 3, 5)])
def test_oracle_full_matches_dense(nx, ny, m):
    z = full_blocks(nx, ny, m, nx * 10 + ny + m)
    o = oracle.Oracle(nx, ny, m, z, layout="full")
    x = gen.rhs_normal(nx * ny * m, 1, 3)[:, 0]
    assert rel(o.applyA(x), dense(nx, ny, m, z) @ x) < 1e-13
    assert np.allclose(o.dense(), dense(nx, ny, m, z), rtol=0, atol=1e-15)


def test_oracle_full_reciprocal_equals_sparse():
    nx, ny, m = 4, 3, 6
    z = full_blocks(nx, ny, m, 5, reciprocal=True)
    of = oracle.Oracle(nx, ny, m, z, layout="full")
    os_ = oracle.Oracle(nx, ny, m, sparse_from_full(nx, ny, z))
    x = gen.rhs_normal(nx * ny * m, 1, 4)[:, 0]
    assert rel(of.applyA(x), os_.applyA(x)) < 1e-14


def _rep(nx, ny, m, seed, corr=True, reciprocal=False):
    base = ToeplitzRep.synthetic(Config("full", nx, ny, m, 1, 4 if corr else -1, seed, "normal", 20,
                                        scale=0.1 if corr else 0.0))
    return ToeplitzRep(nx, ny, m, full_blocks(nx, ny, m, seed, reciprocal), base.correction, None, "full")


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,m,k", [(6, 5, 64, 1), (6, 5, 64, 3), (8, 4, 96, 1), (5, 3, 24, 1), (4, 4, 24, 2),
                                       (32, 32, 64, 1), (7, 2, 40, 1)])
def test_gpu_full_apply(gpu, nx, ny, m, k):
    rep = _rep(nx, ny, m, nx + ny + m)
    op = ToeplitzMatvec(rep, max_nrhs=k)
    o = oracle.Oracle.from_rep(rep)
    X = gen.rhs_normal(o.n, k, 5)
    Y = op.apply(X if k > 1 else X[:, 0]).reshape(o.n, k)
    for c in range(k):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert rel(Y[:, c], ref) < 1e-11, (c, rel(Y[:, c], ref))
    assert np.allclose(op.diagonal(), o.diagonal(), rtol=1e-14, atol=0)


@pytest.mark.gpu
def test_gpu_full_reciprocal_input_is_the_sparse_operator(gpu):
    nx, ny, m = 6, 5, 64
    rep = _rep(nx, ny, m, 7, reciprocal=True)
    sparse = ToeplitzRep(nx, ny, m, sparse_from_full(nx, ny, rep.generators), rep.correction)
    x = gen.rhs_normal(nx * ny * m, 1, 2)[:, 0]
    assert np.array_equal(ToeplitzMatvec(rep).apply(x), ToeplitzMatvec(sparse).apply(x))


@pytest.mark.gpu
def test_gpu_full_gmres(gpu):
    nx, ny, m = 4, 4, 24
    rep = _rep(nx, ny, m, 11)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    b = gen.rhs_normal(o.n, 1, 9)[:, 0]
    g = op.gmres(b, SolverOptions(tol=1e-8, maxIter=300, restart=30), raise_on_fail=False)
    r = o.gmres(b, tol=1e-8, max_iter=300, restart=30)
    assert g.iterations == r["iterations"] and rel(g.current, r["x"]) < 1e-8
    h, hr = g.history[0], r["history"][0]
    assert h.shape == hr.shape and np.all(np.abs(h[:, 1] - hr[:, 1]) <= 1e-8 * np.abs(hr[:, 1]) + 1e-14)
