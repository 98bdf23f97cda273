"""Parity of the non-default product paths selected by environment knobs
(read once per process, so tests/test_env_paths.py runs this script in a
fresh subprocess per setting). Prints "OK <check>" per passed check and
exits non-zero on the first mismatch.

    TBT_APPLY=multi python tests/env_paths_check.py apply gmres
"""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import oracle  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, Config, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check_apply():
    """C2 apply (host buffers) and a 3-column apply against the oracle."""
    cfg = CONFIGS["C2"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep, max_nrhs=3)
    o = oracle.Oracle.from_rep(rep)
    X = gen.rhs_normal(cfg.n, 3, 4)
    Y = op.apply(X)
    for c in range(3):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert rel(Y[:, c], ref) < 1e-11, ("apply", c, rel(Y[:, c], ref))
        assert rel(op.apply(np.ascontiguousarray(X[:, c])), ref) < 1e-11


def check_gmres():
    """C1 to convergence and C2 over a 60-iteration budget (one restart)."""
    for name, budget in (("C1", 2000), ("C2", 60)):
        cfg = CONFIGS[name]
        rep = ToeplitzRep.synthetic(cfg)
        op = ToeplitzMatvec(rep)
        o = oracle.Oracle.from_rep(rep)
        b = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
        g = op.gmres(b, SolverOptions(tol=cfg.tol, maxIter=budget, restart=cfg.restart), raise_on_fail=False)
        r = o.gmres(b, tol=cfg.tol, max_iter=budget, restart=cfg.restart)
        assert g.iterations == r["iterations"], (name, g.iterations, r["iterations"])
        assert rel(g.current, r["x"]) < 1e-8, (name, rel(g.current, r["x"]))
        h, hr = g.history[0], r["history"][0]
        assert h.shape == hr.shape and np.all(np.abs(h[:, 1] - hr[:, 1]) <= 1e-8 * np.abs(hr[:, 1]) + 1e-14)


def check_smooth():
    """C3 grid (18 x 9, smooth 36 x 18 embedding), 8 columns."""
    cfg = Config("s", 18, 9, 64, 8, 8, 3, "normal", 50)
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep, max_nrhs=8, embed="smooth")
    o = oracle.Oracle.from_rep(rep)
    X = gen.rhs_normal(cfg.n, 8, 6)
    Y = op.apply(X)
    for c in range(8):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert rel(Y[:, c], ref) < 1e-11, ("smooth", c)


def check_wide():
    """Wide batches (C3 grid, m = 128, 16 columns: B = 2048), both
    embeddings: register line passes by default, cluster 2-D kernels under
    TBT_FFT=fused."""
    for embed in ("smooth", "pow2"):
        cfg = Config("w", 18, 9, 128, 16, 8, 3, "normal", 50)
        rep = ToeplitzRep.synthetic(cfg)
        op = ToeplitzMatvec(rep, max_nrhs=16, embed=embed)
        o = oracle.Oracle.from_rep(rep)
        X = gen.rhs_normal(cfg.n, 16, 7)
        Y = op.apply(X)
        for c in (0, 5, 15):
            ref = o.apply(np.ascontiguousarray(X[:, c]))
            assert rel(Y[:, c], ref) < 1e-11, ("wide", embed, c)


def check_margin():
    """Margin coupling (B / B^T / C) single- and multi-column."""
    nx, ny, m, e = 4, 3, 6, [2, 3, 1, 4, 6, 2, 3, 5, 1]
    rep = ToeplitzRep.synthetic(Config("mg", nx, ny, m, 1, 2, 3, "normal", 20))
    rep.margin = gen.margin(nx, ny, e, 103)
    op = ToeplitzMatvec(rep, max_nrhs=2)
    o = oracle.Oracle.from_rep(rep)
    X = gen.rhs_normal(o.n, 2, 5)
    Y = op.apply(X)
    for c in range(2):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert rel(Y[:, c], ref) < 1e-11 and rel(op.apply(np.ascontiguousarray(X[:, c])), ref) < 1e-11


def check_dist():
    """Sharded apply + GMRES: one NCCL rank (exchanges to itself, captured in
    a CUDA graph) and three loopback ranks, with the chunk count of the
    overlapped exchanges forced by TBT_DIST_CHUNKS."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2506_04710_b200 import dist_unique_id, loopback_group_id
    for (nx, ny, m), k in (((32, 32, 64), 1), ((6, 5, 64), 3), ((4, 4, 24), 1)):
        rep = ToeplitzRep.synthetic(Config("d", nx, ny, m, 1, 4, 3, "normal", 20))
        o = oracle.Oracle.from_rep(rep)
        X = gen.rhs_normal(o.n, k, 5)
        op = ToeplitzMatvec(rep, max_nrhs=k, dist=(1, 0, dist_unique_id()))
        for _ in range(2):
            Y = op.apply(X if k > 1 else X[:, 0]).reshape(o.n, k)
            for c in range(k):
                assert rel(Y[:, c], o.apply(np.ascontiguousarray(X[:, c]))) < 1e-11, ("nccl", nx, c)
        opt = SolverOptions(tol=1e-8, maxIter=60, restart=15)
        g = op.gmres(X, opt, raise_on_fail=False)
        r = o.gmres(X, tol=1e-8, max_iter=60, restart=15)
        assert g.iterations == r["iterations"], ("nccl gmres", g.iterations, r["iterations"])
        op.close()
        P = 3
        gid = loopback_group_id()
        ops = [ToeplitzMatvec(rep, max_nrhs=k, dist=(P, q, gid, "loopback")) for q in range(P)]
        parts = []
        for q in ops:
            r0, r1 = q.rows()
            parts.append(np.ascontiguousarray(X[r0 * nx * m:r1 * nx * m]))
        with ThreadPoolExecutor(P) as ex:
            Ys = list(ex.map(lambda q: ops[q].apply(parts[q] if k > 1 else parts[q][:, 0]), range(P)))
        Y = np.concatenate([y.reshape(-1, k) for y in Ys], axis=0)
        for c in range(k):
            assert rel(Y[:, c], o.apply(np.ascontiguousarray(X[:, c]))) < 1e-11, ("loopback", nx, c)
        for q in ops:
            q.close()


def check_many():
    """tbt_apply_many over pinned and pageable C2 batches: bit-identical to
    single applies, oracle parity on the first and last vector."""
    import torch
    cfg = CONFIGS["C2"]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    X = np.ascontiguousarray(gen.rhs_normal(cfg.n, 5, 9).T)
    xt = torch.from_numpy(X.copy()).pin_memory()
    yt = torch.empty_like(xt).pin_memory()
    op.apply_many_ptr(xt.data_ptr(), yt.data_ptr(), 5)
    for Y in (yt.numpy(), op.apply_many(X)):
        for i in range(5):
            assert np.array_equal(Y[i], op.apply(X[i])), ("many", i)
        for i in (0, 4):
            assert rel(Y[i], o.apply(X[i])) < 1e-11, ("many oracle", i)


CHECKS = {"apply": check_apply, "many": check_many, "gmres": check_gmres, "smooth": check_smooth, "margin": check_margin,
          "wide": check_wide, "dist": check_dist}

if __name__ == "__main__":
    for name in sys.argv[1:]:
        CHECKS[name]()
        print("OK", name, flush=True)
