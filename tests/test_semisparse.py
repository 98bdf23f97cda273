"""SemiSparse representations (reference ToeplitzRep::aLevel1 + bFull +
cFull, toeplitz.hpp:90-93).

The reference's SemiSparse ToeplitzMatvec runs the same FFT applyA with
generators read out of aLevel1 (aEntry, linsolve.cpp:220-224) and applies
B, B^T and C as dense products (:294, :318, :338). Here: a SemiSparse ZTOE1
cache is written from a Sparse operator's dense matrix, with the aLevel1
blocks aEntry never reads filled with noise (both sides must ignore them),
then parsed (csrc/io.cu), run through the oracle (CPU) and the CUDA path
(GPU), and compared with the reference itself reading the same file."""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import (DenseMargin, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen,
                                   generators_from_level1, read_ztoe1)
from test_ref_pin import margin_case, needs_ref, rel
from ztoe1_writer import write_ztoe1_dense

CASES = [(3, 3, 4, [1, 2, 1, 2, 4, 1, 1, 2, 1]), (4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]),
         (5, 2, 3, [0, 2, 0, 1, 3, 0, 1, 0, 2]), (3, 4, 5, [0] * 4 + [5] + [0] * 4)]


def semisparse_file(tmp_path, nx, ny, m, e, seed=4):
    """(path, dense Z, generators) of a SemiSparse cache equal to a Sparse
    operator, with the aLevel1 blocks outside aEntry's reach randomised."""
    g = gen.blocks_raw(nx, ny, m, seed)
    if sum(e) == e[4]:
        from ztoe1_writer import write_ztoe1
        p = tmp_path / "a.ztoe1"
        write_ztoe1(str(p), nx, ny, e, g)
        Z = oracle.Oracle(nx, ny, m, g).dense()
    else:
        R, O, _ = margin_case(tmp_path, nx, ny, m, e, seed)
        Z = R.dense()
    nA = nx * ny * m
    rng = np.random.default_rng(seed + 1)
    a1 = []
    for i in range(ny):
        blk = Z[i * nx * m:(i + 1) * nx * m, 0:nx * m].copy()
        for c1 in range(nx):
            for c2 in range(nx):
                if not (c2 == 0 or c1 == 0):  # (max(j,0), max(-j,0)) always has a zero index
                    blk[c1 * m:(c1 + 1) * m, c2 * m:(c2 + 1) * m] = rng.standard_normal((m, m))
        a1.append(blk)
    path = tmp_path / f"semi_{nx}_{ny}_{m}.ztoe1"
    write_ztoe1_dense(str(path), nx, ny, e, 1, a_level1=a1, b_full=Z[nA:, :nA], c_full=Z[nA:, nA:])
    return path, Z, g, a1


@pytest.mark.parametrize("nx,ny,m,e", CASES)
def test_parse_semisparse(tmp_path, nx, ny, m, e):
    path, Z, g, a1 = semisparse_file(tmp_path, nx, ny, m, e)
    rep = read_ztoe1(str(path))
    assert np.array_equal(rep.generators, g)
    assert np.array_equal(generators_from_level1(nx, ny, m, a1), g)
    nA = nx * ny * m
    if nA == Z.shape[0]:
        assert rep.margin is None
        return
    assert isinstance(rep.margin, DenseMargin)
    nM = Z.shape[0] - nA
    assert np.array_equal(rep.margin.b_full.reshape(nA, nM).T, Z[nA:, :nA])
    assert np.array_equal(rep.margin.c.reshape(nM, nM).T, Z[nA:, nA:])


@needs_ref
@pytest.mark.parametrize("nx,ny,m,e", CASES)
def test_oracle_semisparse_matches_reference(tmp_path, nx, ny, m, e):
    path, Z, g, _ = semisparse_file(tmp_path, nx, ny, m, e)
    R = oracle.RefOperator(path)
    assert R.mode == 1
    O = oracle.Oracle.from_rep(read_ztoe1(str(path)))
    x = gen.rhs_normal(R.n, 1, 5)[:, 0]
    assert rel(O.apply(x), R.apply(x)) <= 1e-14
    assert np.array_equal(O.diagonal(), R.diagonal())
    if R.nM:
        b = gen.rhs_normal(R.n, 1, 9)[:, 0]
        r = R.gmres(b, tol=1e-8, max_iter=300, restart=30)
        o = O.gmres(b, tol=1e-8, max_iter=300, restart=30)
        assert r["iterations"] == o["iterations"][0] and rel(o["x"], r["x"]) <= 1e-12


def test_full_mode_cache_rejected(tmp_path):
    from paper_2506_04710_b200 import UserError
    p = tmp_path / "full.ztoe1"
    write_ztoe1_dense(str(p), 2, 2, [0] * 4 + [2] + [0] * 4, 0, z_full=np.eye(8, dtype=complex))
    with pytest.raises(UserError, match="Full-mode"):
        read_ztoe1(str(p))


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,m,e", CASES[:3])
def test_gpu_semisparse_matches_reference(gpu, tmp_path, nx, ny, m, e):
    path, Z, g, _ = semisparse_file(tmp_path, nx, ny, m, e)
    R = oracle.RefOperator(path)
    for op in (ToeplitzMatvec.from_ztoe1(str(path), max_nrhs=2), ToeplitzMatvec(read_ztoe1(str(path)), max_nrhs=2)):
        X = gen.rhs_normal(R.n, 2, 5)
        Y = op.apply(X)
        for c in range(2):
            assert rel(Y[:, c], R.apply(np.ascontiguousarray(X[:, c]))) <= 1e-11
        x = np.ascontiguousarray(X[:, 0])
        assert rel(op.applyB(x[:R.nA]), R.applyB(x[:R.nA])) <= 1e-11
        assert rel(op.applyBT(x[R.nA:]), R.applyBT(x[R.nA:])) <= 1e-11
        assert rel(op.applyC(x[R.nA:]), R.applyC(x[R.nA:])) <= 1e-11
        assert np.array_equal(op.diagonal(), R.diagonal())
        b = gen.rhs_normal(R.n, 1, 9)[:, 0]
        r = R.gmres(b, tol=1e-8, max_iter=300, restart=30)
        res = op.gmres(b, SolverOptions(tol=1e-8, maxIter=300, restart=30), raise_on_fail=False)
        assert res.iterations[0] == r["iterations"] and rel(res.current, r["x"]) <= 1e-8
        V = np.zeros((R.n, 2), complex)
        V[:R.nA] = gen.rhs_normal(R.nA, 2, 10)
        rs = R.solve("schur", V, tol=1e-10, restart=30)
        ss = op.schur_solve(V, SolverOptions(tol=1e-10, maxIter=2000, restart=30))
        assert ss.iterations == rs["iterations"] and rel(ss.current, rs["x"]) <= 1e-8
        op.close()
