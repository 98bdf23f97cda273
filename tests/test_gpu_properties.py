"""SPEC.md's hot-path known-answer properties, checked on the
CUDA path itself through the C ABI — at full BASELINE sizes where the
property is size-independent (no oracle run needed there):

* x = 0 gives y = 0 exactly; linearity to < 1e-12;
* the operator is symmetric for reciprocal generators, u^T (Z v) = (Z u)^T v
  (A(-s) = A(s)^T, linsolve.cpp:219; the edge/corner terms add P and P^T);
* applies are deterministic (fixed-order reductions: bitwise repeatable);
* a batched apply over 50 random vectors matches the dense product < 1e-12
  (dense Z = the oracle's assembly, C1 N = 384);
* GMRES on V = Z e_1 recovers e_1; Jacobi never needs more iterations than
  the unpreconditioned solve; iterative and dense solves
  agree < 1e-8.
"""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def cvec(n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


@pytest.fixture(scope="module")
def ops(gpu):
    made = {}

    def get(name):
        if name not in made:
            made[name] = ToeplitzMatvec(ToeplitzRep.synthetic(CONFIGS[name]), max_nrhs=50 if name == "C1" else 1)
        return made[name]

    yield get
    for op in made.values():
        op.close()


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_zero_linearity_symmetry_determinism(ops, name):
    op = ops(name)
    n = op.size()
    assert not np.any(op.apply(np.zeros(n, complex)))  # exact zeros
    x, w = cvec(n, 1), cvec(n, 2)
    a, b = 0.3 - 1.2j, 2.0 + 0.5j
    zx, zw = op.apply(x), op.apply(w)
    assert rel(op.apply(a * x + b * w), a * zx + b * zw) < 1e-12
    # Reciprocity: x^T Z w == (Z x)^T w (bilinear, no conjugation).
    lhs, rhs = x @ zw, zx @ w
    assert abs(lhs - rhs) / (np.linalg.norm(x) * np.linalg.norm(zw)) < 1e-13
    # Fixed-order reductions: the same input gives the same bits.
    assert np.array_equal(op.apply(x).view(np.uint64), zx.view(np.uint64))


def test_dense_50_vectors_c1(ops):
    op = ops("C1")
    o = oracle.Oracle.from_rep(ToeplitzRep.synthetic(CONFIGS["C1"]))
    Z = o.dense()
    rng = np.random.default_rng(7)
    X = rng.standard_normal((o.n, 50)) + 1j * rng.standard_normal((o.n, 50))
    Y = op.apply(X)
    Yd = Z @ X
    for c in range(50):  # SPEC.md:448, per vector
        assert rel(Y[:, c], Yd[:, c]) < 1e-12, c


def test_gmres_recovers_unit_vector_and_dense_agreement(ops):
    cfg = CONFIGS["C1"]
    op = ops("C1")
    o = oracle.Oracle.from_rep(ToeplitzRep.synthetic(cfg))
    Z = o.dense()
    e1 = np.zeros(o.n, complex)
    e1[0] = 1.0
    r = op.gmres(Z @ e1, SolverOptions(tol=1e-10, maxIter=cfg.max_iter, restart=cfg.restart))
    assert r.converged[0] and np.linalg.norm(r.current - e1) < 1e-8
    b = cvec(o.n, 11)
    r = op.gmres(b, SolverOptions(tol=1e-10, maxIter=cfg.max_iter, restart=cfg.restart))
    assert rel(r.current, np.linalg.solve(Z, b)) < 1e-8


def test_jacobi_not_worse(ops):
    cfg = CONFIGS["C1"]
    op = ops("C1")
    b = cvec(op.size(), 12)
    its = []
    for pre in (True, False):
        r = op.gmres(b, SolverOptions(tol=cfg.tol, maxIter=cfg.max_iter, restart=cfg.restart, precondition=pre))
        assert r.converged[0]
        its.append(r.iterations[0])
    assert its[0] <= its[1], its
