"""tbt_apply_many: a batch of independent single-column vectors in host
memory, host copies overlapped with the applies (csrc/api.cu). Every
result must be bit-identical to tbt_apply on the same vector (same kernels,
same order), and match the oracle (reference applyA + correction,
linsolve.cpp:260-290) at 1e-11; pinned and pageable buffers; the FULL
layout (multi-launch path); empty batches; margin contexts are a user
error."""
import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import CONFIGS, Config, ToeplitzMatvec, ToeplitzRep, UserError, gen

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,count", [("C1", 1), ("C1", 5), ("C2", 7)])
def test_apply_many_matches_apply(gpu, name, count):
    cfg = CONFIGS[name]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    X = np.ascontiguousarray(gen.rhs_normal(cfg.n, count, 21).T)  # (count, n)
    Y = op.apply_many(X)
    o = oracle.Oracle.from_rep(rep)
    for i in range(count):
        assert np.array_equal(Y[i], op.apply(X[i])), i
    for i in {0, count - 1}:
        assert rel(Y[i], o.apply(X[i])) < 1e-11


def test_apply_many_pinned(gpu):
    import torch
    cfg = CONFIGS["C2"]
    op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg))
    X = np.ascontiguousarray(gen.rhs_normal(cfg.n, 9, 22).T)
    xt = torch.from_numpy(X.copy()).pin_memory()
    yt = torch.empty_like(xt).pin_memory()
    for _ in range(2):  # slots reused across calls
        op.apply_many_ptr(xt.data_ptr(), yt.data_ptr(), 9)
        Y = yt.numpy()
        for i in (0, 4, 8):
            assert np.array_equal(Y[i], op.apply(X[i]))


@pytest.mark.parametrize("count", [1, 2, 3, 16])
def test_apply_many_pinned_every_vector(gpu, count):
    """Pinned batches (two device slots per direction, copies on both copy
    engines): every vector, first and last included, is bit-identical to a
    single device-resident apply."""
    import torch
    cfg = CONFIGS["C2"]
    op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg))
    X = np.ascontiguousarray(gen.rhs_normal(cfg.n, count, 40 + count).T)
    xt = torch.from_numpy(X.copy()).pin_memory()
    yt = torch.full_like(xt, complex("nan")).pin_memory()
    op.apply_many_ptr(xt.data_ptr(), yt.data_ptr(), count)
    Y = yt.numpy()
    for i in range(count):
        assert np.array_equal(Y[i], op.apply(X[i])), i


def test_apply_many_full_layout_and_edges(gpu):
    from test_full_layout import _rep
    rep = _rep(5, 3, 24, 4)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    X = np.ascontiguousarray(gen.rhs_normal(o.n, 3, 23).T)
    Y = op.apply_many(X)
    for i in range(3):
        assert rel(Y[i], o.apply(X[i])) < 1e-11
    assert op.apply_many(np.empty((0, o.n), complex)).shape == (0, o.n)
    with pytest.raises(ValueError):
        op.apply_many(np.zeros((2, o.n + 1), complex))


def test_apply_many_rejects_margin(gpu):
    nx, ny, m, e = 4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]
    rep = ToeplitzRep.synthetic(Config("mg", nx, ny, m, 1, 2, 3, "normal", 20))
    rep.margin = gen.margin(nx, ny, e, 103)
    op = ToeplitzMatvec(rep)
    with pytest.raises(UserError):
        op.apply_many(np.zeros((2, op.size()), complex))
