"""Multi-GPU partition (csrc/dist.cu).

CPU: the partition (tbt_dist_plan) covers rows and bin columns exactly once
with column groups closed under s0 -> L0 - s0; a 2-process gloo run executes
the sharded algorithm (row FFTs, all-to-all, column FFTs, per-rank bin
products, the transposes back) with that partition in numpy and must equal
the oracle's apply. GPU (1 device here): the NCCL path with a one-rank
communicator through the C ABI against the oracle."""
import os
import socket

import numpy as np
import pytest

from paper_2506_04710_b200 import Config, ToeplitzRep, dist_plan

SHAPES = [(32, 64, 1), (32, 64, 2), (32, 64, 3), (32, 64, 8), (9, 36, 4), (9, 32, 8), (4, 8, 2), (1, 1, 1),
          (3, 9, 2), (64, 128, 8)]


@pytest.mark.parametrize("ny,L0,P", SHAPES)
def test_plan_partitions(ny, L0, P):
    rows, cols = [], []
    for r in range(P):
        r0, r1, c = dist_plan(ny, L0, P, r)
        rows.append((r0, r1))
        cols.append(c)
        assert c == sorted(c)
        for s in c:  # closed under negation: both bins of every pair are local
            assert (L0 - s) % L0 in c
    assert rows[0][0] == 0 and rows[-1][1] == ny
    assert all(rows[k][1] == rows[k + 1][0] for k in range(P - 1))
    assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1
    flat = sorted(s for c in cols for s in c)
    assert flat == list(range(L0))
    if L0 >= 2 * P:
        sizes = [len(c) for c in cols]
        assert max(sizes) - min(sizes) <= 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nx, ny, m, q):
    import torch
    import torch.distributed as tdist

    import oracle
    from paper_2506_04710_b200 import gen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Config("d", nx, ny, m, 1, 4, 7, "normal", 20)
        rep = ToeplitzRep.synthetic(cfg)
        o = oracle.Oracle.from_rep(rep)
        ah = o.ahat()  # [a][b][f] (test-side spectrum)
        L0, L1 = o.bins and (1 << (2 * nx - 2).bit_length()), 1 << (2 * ny - 2).bit_length()
        L = L0 * L1
        plan = [dist_plan(ny, L0, world, r) for r in range(world)]
        r0, r1, mycols = plan[rank]
        x = gen.rhs_normal(o.n, 1, 11)[:, 0]
        xg = x.reshape(ny, nx, m)
        # 1. row FFTs of my rows
        trow = np.fft.fft(xg[r0:r1], n=L0, axis=1)  # [r][s0][a]
        # 2. all-to-all: my rows x columns of q -> q
        send = np.concatenate([trow[:, plan[q][2], :].ravel() for q in range(world)])
        scount = [(r1 - r0) * len(plan[q][2]) * m for q in range(world)]
        rcount = [(plan[q][1] - plan[q][0]) * len(mycols) * m for q in range(world)]
        recv = torch.empty(sum(rcount), dtype=torch.complex128)
        tdist.all_to_all_single(recv, torch.from_numpy(send), rcount, scount)
        tcol = recv.numpy().reshape(ny, len(mycols), m)  # rank slabs ordered -> all rows
        # 3. column FFTs of my columns
        xh = np.fft.fft(tcol, n=L1, axis=0)  # [s1][j][a]
        # 4. bin products on my bins
        yh = np.zeros_like(xh)
        for s1 in range(L1):
            for j, s0 in enumerate(mycols):
                yh[s1, j] = ah[:, :, s1 * L0 + s0] @ xh[s1, j]
        # 5. inverse column FFTs, keep ny rows; all-to-all back
        tc = np.fft.ifft(yh, axis=0)[:ny] * L1  # unscaled inverse
        send2 = np.concatenate([tc[plan[q][0]:plan[q][1]].ravel() for q in range(world)])
        s2 = [(plan[q][1] - plan[q][0]) * len(mycols) * m for q in range(world)]
        r2 = [(r1 - r0) * len(plan[q][2]) * m for q in range(world)]
        recv2 = torch.empty(sum(r2), dtype=torch.complex128)
        tdist.all_to_all_single(recv2, torch.from_numpy(send2), r2, s2)
        trow2 = np.zeros((r1 - r0, L0, m), dtype=complex)
        off = 0
        for qq in range(world):
            nq = len(plan[qq][2])
            blk = recv2.numpy()[off:off + (r1 - r0) * nq * m].reshape(r1 - r0, nq, m)
            trow2[:, plan[qq][2], :] = blk
            off += (r1 - r0) * nq * m
        # 6. inverse row FFTs, keep nx, 1/L
        y = (np.fft.ifft(trow2, axis=1)[:, :nx] * L0) / L
        ref = o.applyA(x).reshape(ny, nx, m)[r0:r1]
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        q.put((rank, float(err)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("nx,ny,m", [(5, 6, 4), (8, 3, 6)])
def test_sharded_algorithm_gloo_two_ranks(nx, ny, m):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nx, ny, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    errs = dict(q.get(timeout=10) for _ in range(2))
    assert set(errs) == {0, 1}
    assert max(errs.values()) < 1e-12, errs


@pytest.mark.gpu
@pytest.mark.parametrize("shape,embed,k", [((4, 4, 24), "pow2", 1), ((32, 32, 64), "pow2", 1),
                                           ((18, 9, 8), "smooth", 1), ((6, 5, 64), "pow2", 3)])
def test_dist_one_rank_nccl(gpu, shape, embed, k):
    import oracle
    from paper_2506_04710_b200 import ToeplitzMatvec, dist_unique_id, gen
    nx, ny, m = shape
    rep = ToeplitzRep.synthetic(Config("d", nx, ny, m, 1, 4, 3, "normal", 20))
    op = ToeplitzMatvec(rep, max_nrhs=k, embed=embed, dist=(1, 0, dist_unique_id()))
    assert op.info().apply_path == 3 and op.rows() == (0, ny)
    o = oracle.Oracle.from_rep(rep)
    X = gen.rhs_normal(o.n, k, 5)
    Y = op.apply(X if k > 1 else X[:, 0])
    Y = Y.reshape(o.n, k)
    for c in range(k):
        ref = o.apply(np.ascontiguousarray(X[:, c]))
        assert np.linalg.norm(Y[:, c] - ref) / np.linalg.norm(ref) < 1e-11
    assert np.allclose(op.diagonal(), o.diagonal(), rtol=1e-14, atol=0)


def _ls_gmres_worker(rank, world, port, q, tol, max_iter, restart):
    """Distributed GMRES as the column-blocked CUDA path runs it
    (csrc/gmres.cu, ColsRunner): element-row slabs, every reduction a local
    partial + all_reduce, low-synchronisation MGS h = (I + L)^{-1} V^H M w,
    Givens / restart / history rules of linsolve.cpp:425-515."""
    import torch
    import torch.distributed as tdist

    import oracle
    from paper_2506_04710_b200 import gen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Config("g", 5, 6, 4, 1, 4, 9, "normal", 20)
        rep = ToeplitzRep.synthetic(cfg)
        o = oracle.Oracle.from_rep(rep)
        L0 = 1 << (2 * cfg.nx - 2).bit_length()
        r0, r1, _ = dist_plan(cfg.ny, L0, world, rank)
        sl = slice(r0 * cfg.nx * cfg.m, r1 * cfg.nx * cfg.m)
        b = gen.rhs_normal(o.n, 1, 13)[:, 0]
        d = o.diagonal()
        dinv = np.where(np.abs(d) > 0, 1.0 / np.where(d == 0, 1, d), 1.0)[sl]
        bl = b[sl]

        def allsum(a):
            t = torch.from_numpy(np.ascontiguousarray(np.atleast_1d(a)))
            tdist.all_reduce(t)
            return t.numpy()

        def matvec(xl):
            parts = [torch.zeros(0, dtype=torch.complex128) for _ in range(world)]
            tdist.all_gather_object(parts, xl)
            return o.apply(np.concatenate(parts))[sl]

        def nrm(v):
            return float(np.sqrt(allsum(np.array([np.vdot(v, v).real]))[0]))

        bnorm = nrm(bl)
        x = np.zeros_like(bl)
        hist, its, beta0 = [], 0, 0.0
        while True:
            r = bl - matvec(x)
            res = nrm(r) / bnorm
            if res < tol:
                hist.append((0.0, res))
                break
            if its >= max_iter:
                hist.append((2.0, res))
                break
            hist.append((0.0, res))
            z = dinv * r
            beta = nrm(z)
            beta0 = beta0 or beta
            V = [z / beta]
            H = np.zeros((restart + 1, restart), complex)
            S = np.zeros((restart + 1, restart + 1), complex)
            cs, sn = np.zeros(restart, complex), np.zeros(restart, complex)
            g = np.zeros(restart + 1, complex)
            g[0] = beta
            nc = 0
            for j in range(restart):
                wz = dinv * matvec(V[j])
                loc = np.array([np.vdot(V[k], wz) for k in range(j + 1)] + [np.vdot(V[j], V[k]) for k in range(j)])
                tot = allsum(loc)
                c, S[j, :j] = tot[:j + 1], tot[j + 1:]
                h = c.copy()
                for k in range(j):
                    h[k + 1:] -= S[k + 1:j + 1, k] * h[k]
                w = wz - sum(h[k] * V[k] for k in range(j + 1))
                hn = nrm(w)
                if hn > 0:
                    V.append(w / hn)
                col = np.zeros(restart + 1, complex)
                col[:j + 1], col[j + 1] = h, hn
                for i in range(j):
                    a0, a1 = col[i], col[i + 1]
                    col[i] = cs[i] * a0 + sn[i] * a1
                    col[i + 1] = -np.conj(sn[i]) * a0 + np.conj(cs[i]) * a1
                den = np.sqrt(abs(col[j]) ** 2 + abs(col[j + 1]) ** 2)
                cs[j], sn[j] = (1, 0) if den == 0 else (np.conj(col[j]) / den, np.conj(col[j + 1]) / den)
                col[j] = cs[j] * col[j] + sn[j] * col[j + 1]
                col[j + 1] = 0
                H[:, j] = col
                g[j + 1] = -np.conj(sn[j]) * g[j]
                g[j] = cs[j] * g[j]
                its += 1
                nc = j + 1
                hist.append((1.0, abs(g[j + 1]) / beta0))
                if abs(g[j + 1]) / beta < 0.1 * tol or not hn > 0 or its >= max_iter:
                    break
            y = np.zeros(nc, complex)
            for i in range(nc - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:nc] @ y[i + 1:nc]) / H[i, i]
            x = x + sum(y[i] * V[i] for i in range(nc))
        ref = o.gmres(b, tol=tol, max_iter=max_iter, restart=restart)
        herr = max(abs(a[1] - bb[1]) / max(abs(bb[1]), 1e-300) for a, bb in zip(hist, ref["history"][0]))
        kinds_ok = [a[0] for a in hist] == [float(v) for v in ref["history"][0][:, 0]]
        xerr = np.linalg.norm(x - ref["x"][sl]) / np.linalg.norm(ref["x"][sl])
        q.put((rank, its == ref["iterations"][0], kinds_ok, float(herr), float(xerr)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("tol,max_iter,restart", [(1e-9, 400, 10), (1e-12, 23, 7)])
def test_distributed_ls_gmres_gloo_two_ranks(tol, max_iter, restart):
    """The multi-GPU solve's algorithm on 2 gloo ranks equals the oracle's
    (MGS) GMRES: iteration count, history kinds and values, solution."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ls_gmres_worker, args=(r, 2, port, q, tol, max_iter, restart)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    out = [q.get(timeout=10) for _ in range(2)]
    for rank, its_ok, kinds_ok, herr, xerr in out:
        assert its_ok and kinds_ok, out
        assert herr < 1e-8 and xerr < 1e-8, out


@pytest.mark.gpu
@pytest.mark.parametrize("shape,k", [((4, 4, 24), 1), ((6, 5, 64), 3), ((4, 3, 128), 12)])
def test_dist_gmres_one_rank_nccl(gpu, shape, k):
    """tbt_gmres on a distributed context (column-blocked kernels, NCCL
    all-reduces on a one-rank communicator) against the oracle."""
    import oracle
    from paper_2506_04710_b200 import SolverOptions, ToeplitzMatvec, dist_unique_id, gen
    nx, ny, m = shape
    rep = ToeplitzRep.synthetic(Config("d", nx, ny, m, 1, 4, 3, "normal", 20))
    op = ToeplitzMatvec(rep, max_nrhs=k, dist=(1, 0, dist_unique_id()))
    o = oracle.Oracle.from_rep(rep)
    B = gen.rhs_normal(o.n, k, 9)
    g = op.gmres(B, SolverOptions(tol=1e-8, maxIter=120, restart=15), raise_on_fail=False)
    r = o.gmres(B, tol=1e-8, max_iter=120, restart=15)
    assert g.iterations == r["iterations"] and g.converged == r["converged"]
    for c in range(k):
        assert np.linalg.norm(g.current[:, c] - r["x"][:, c]) / np.linalg.norm(r["x"][:, c]) < 1e-8
        h, hr = g.history[c], r["history"][c]
        assert h.shape == hr.shape and np.array_equal(h[:, 0], hr[:, 0])
        assert np.all(np.abs(h[:, 1] - hr[:, 1]) <= 1e-8 * np.abs(hr[:, 1]) + 1e-14)
