"""The sharded operator at P > 1 on ONE GPU.

P rank contexts of this process share an in-process loopback transport
(tbt_dist_init_loopback): each rank runs the exact pack / exchange / unpack
code of the NCCL path (csrc/dist.cu) and the distributed GMRES all-reduces
(csrc/gmres.cu), from its own host thread; exchanges synchronise the rank's
stream, meet at a host barrier and copy device to device, so no kernel ever
waits on another rank. The concatenated row slabs must match the oracle
(matvec <= 1e-11; GMRES iteration counts identical, solution and residual
history within 1e-8). The reference has no counterpart: this replaces its
per-column parallelFor (proj/src/linsolve.cpp:572)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_2506_04710_b200 import Config, SolverOptions, ToeplitzMatvec, ToeplitzRep, UserError, gen
from paper_2506_04710_b200 import loopback_group_id

pytestmark = pytest.mark.gpu


def make_group(rep, P, k=1, embed="pow2"):
    gid = loopback_group_id()
    return [ToeplitzMatvec(rep, max_nrhs=k, embed=embed, dist=(P, r, gid, "loopback")) for r in range(P)]


def on_ranks(ops, fn):
    """fn(rank, op) on every rank concurrently (one host thread per rank)."""
    with ThreadPoolExecutor(len(ops)) as ex:
        futs = [ex.submit(fn, r, op) for r, op in enumerate(ops)]
        return [f.result(timeout=300) for f in futs]


def slabs(ops, nx, m, X):
    out = []
    for op in ops:
        r0, r1 = op.rows()
        out.append(np.ascontiguousarray(X[r0 * nx * m:r1 * nx * m]))
    return out


def close(ops):
    for op in ops:
        op.close()


APPLY_CASES = [((4, 4, 24), "pow2", 1, P) for P in (2, 3, 4)] + \
              [((32, 32, 64), "pow2", 1, P) for P in (2, 3, 4, 8)] + \
              [((18, 9, 32), "smooth", 1, P) for P in (2, 3, 4, 8)] + \
              [((6, 5, 64), "pow2", 3, P) for P in (2, 3, 4)] + \
              [((20, 16, 24), "pow2", 2, 8)]


@pytest.mark.parametrize("shape,embed,k,P", APPLY_CASES)
def test_loopback_apply(gpu, shape, embed, k, P):
    nx, ny, m = shape
    rep = ToeplitzRep.synthetic(Config("lb", nx, ny, m, 1, 4, 3, "normal", 20))
    ops = make_group(rep, P, k, embed)
    try:
        from paper_2506_04710_b200._lib import lib
        import ctypes as C
        kind = C.c_int()
        lib().tbt_dist_transport(ops[0]._h, C.byref(kind))
        assert kind.value == 2 and ops[0].info().apply_path == 3
        rows = [op.rows() for op in ops]
        assert rows[0][0] == 0 and rows[-1][1] == ny and all(b > a for a, b in rows)
        o = oracle.Oracle.from_rep(rep)
        X = gen.rhs_normal(o.n, k, 5)
        parts = slabs(ops, nx, m, X)
        Y = on_ranks(ops, lambda r, op: op.apply(parts[r] if k > 1 else parts[r][:, 0]))
        Y = np.concatenate([y.reshape(-1, k) for y in Y], axis=0)
        for c in range(k):
            ref = o.apply(np.ascontiguousarray(X[:, c]))
            assert np.linalg.norm(Y[:, c] - ref) / np.linalg.norm(ref) < 1e-11, (P, c)
        # A x without the correction, and the diagonal, slab by slab
        YA = on_ranks(ops, lambda r, op: op.applyA(parts[r][:, 0]))
        refA = o.applyA(np.ascontiguousarray(X[:, 0]))
        assert np.linalg.norm(np.concatenate(YA) - refA) / np.linalg.norm(refA) < 1e-11
        d = np.concatenate([op.diagonal() for op in ops])
        assert np.allclose(d, o.diagonal(), rtol=1e-14, atol=0)
    finally:
        close(ops)


@pytest.mark.parametrize("shape,k,P", [((4, 4, 24), 1, 2), ((4, 4, 24), 1, 4), ((6, 5, 64), 3, 2),
                                       ((6, 5, 64), 3, 4), ((16, 8, 32), 1, 8)])
def test_loopback_gmres(gpu, shape, k, P):
    """Distributed GMRES (column-blocked low-sync Arnoldi, two all-reduces
    per iteration) on P ranks against the oracle's gmres
    (linsolve.cpp:425-515); every rank returns the same stats."""
    nx, ny, m = shape
    rep = ToeplitzRep.synthetic(Config("lb", nx, ny, m, 1, 4, 3, "normal", 20))
    ops = make_group(rep, P, k)
    try:
        o = oracle.Oracle.from_rep(rep)
        B = gen.rhs_normal(o.n, k, 9)
        parts = slabs(ops, nx, m, B)
        opt = SolverOptions(tol=1e-8, maxIter=120, restart=15)
        res = on_ranks(ops, lambda r, op: op.gmres(parts[r], opt, raise_on_fail=False))
        r = o.gmres(B, tol=1e-8, max_iter=120, restart=15)
        for g in res:
            assert g.iterations == r["iterations"] and g.converged == r["converged"]
            assert g.matvecs == res[0].matvecs
        X = np.concatenate([g.current.reshape(-1, k) for g in res], axis=0)
        for c in range(k):
            assert np.linalg.norm(X[:, c] - r["x"][:, c]) / np.linalg.norm(r["x"][:, c]) < 1e-8
            for g in res:
                h, hr = g.history[c], r["history"][c]
                assert h.shape == hr.shape and np.array_equal(h[:, 0], hr[:, 0])
                assert np.all(np.abs(h[:, 1] - hr[:, 1]) <= 1e-8 * np.abs(hr[:, 1]) + 1e-14)
    finally:
        close(ops)


def test_loopback_rejects_more_ranks_than_rows(gpu):
    rep = ToeplitzRep.synthetic(Config("lb", 8, 4, 8, 1, 4, 3, "normal", 20))
    gid = loopback_group_id()
    with pytest.raises(UserError, match="element rows"):
        ToeplitzMatvec(rep, dist=(5, 0, gid, "loopback"))


def test_loopback_failure_releases_the_group(gpu):
    """A rank that fails inside the library aborts the group: the other
    ranks raise instead of waiting at the next exchange."""
    rep = ToeplitzRep.synthetic(Config("lb", 8, 6, 16, 1, 4, 3, "normal", 20))
    ops = make_group(rep, 3, 1)
    try:
        x = gen.rhs_normal(8 * 6 * 16, 2, 1)
        parts = slabs(ops, 8, 16, x)

        def call(r, op):
            try:
                # rank 1 asks for 2 columns on a max_nrhs = 1 context
                op.apply(parts[r] if r == 1 else parts[r][:, 0])
                return "ok"
            except Exception as exc:  # noqa: BLE001
                return type(exc).__name__

        out = on_ranks(ops, call)
        assert out[1] == "UserError" and all(v != "ok" for v in out)
    finally:
        close(ops)
