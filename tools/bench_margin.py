"""Row f1 measurement: the full operator with margin parts (B / B^T / C) on
a BASELINE grid, device-resident, vs the same operator without margin and
vs the oracle on one host core.

    python tools/bench_margin.py [--config C2] [--edges 8]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402
from paper_2506_04710_b200._lib import TBT_DEVICE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--edges", type=int, default=8)
ap.add_argument("--no-cpu", action="store_true")
ap.add_argument("--schur", action="store_true", help="also time schurSolve (needs a config whose A-solves converge, e.g. C1)")
ap.add_argument("--schur-batch", type=int, default=0, help="max_nrhs of the Schur context (default: all inner columns)")
args = ap.parse_args()
cfg = CONFIGS[args.config]
e = [args.edges] * 9
e[4] = cfg.m
rep = ToeplitzRep.synthetic(cfg)
rep.margin = gen.margin(cfg.nx, cfg.ny, e, cfg.seed + 7)
stream = torch.cuda.Stream()
out = {"config": cfg.name, "edges_per_margin_part": args.edges, "nA": cfg.n, "nM": rep.margin.size(cfg.nx, cfg.ny)}


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / n


op = ToeplitzMatvec(rep)
op.set_stream(stream.cuda_stream)
N = op.size()
x = torch.from_numpy(gen.rhs_normal(N, 1, 3)[:, 0].copy()).cuda()
y = torch.empty_like(x)
with torch.cuda.stream(stream):
    for _ in range(5):
        op.apply_device(x.data_ptr(), y.data_ptr())
    out["full_apply_us"] = 1e3 * timed(lambda: op.apply_device(x.data_ptr(), y.data_ptr()), 200)
    out["a_only_apply_us"] = 1e3 * timed(lambda: op.apply_device(x.data_ptr(), y.data_ptr(), a_only=True), 200)
    b = torch.from_numpy(gen.rhs_normal(N, 1, 9)[:, 0].copy()).cuda()
    xs = torch.empty_like(b)
    opt = SolverOptions(tol=1e-8, maxIter=100, restart=50)
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g = op.gmres(None, opt, raise_on_fail=False, where=TBT_DEVICE, b_ptr=b.data_ptr(), x_ptr=xs.data_ptr(), nrhs=1)
        e1.record(stream)
        e1.synchronize()
    out["gmres_ms_per_iteration"] = e0.elapsed_time(e1) / max(g.iterations[0], 1)
    out["gmres_iterations"] = g.iterations[0]
if not args.no_cpu:
    import oracle
    o = oracle.Oracle.from_rep(rep)
    xh = gen.rhs_normal(N, 1, 3)[:, 0]
    o.apply(xh)
    t0, cnt = time.perf_counter(), 0
    while time.perf_counter() - t0 < 5.0 or cnt < 2:
        o.apply(xh)
        cnt += 1
    out["cpu_oracle_full_apply_ms"] = 1e3 * (time.perf_counter() - t0) / cnt
    with torch.cuda.stream(stream):
        op.apply_device(x.data_ptr(), y.data_ptr())
    stream.synchronize()
    yd = y.cpu().numpy()
    ref = o.apply(x.cpu().numpy())
    out["parity_rel_err"] = float(np.linalg.norm(yd - ref) / np.linalg.norm(ref))
if args.schur:
    rep.correction = None  # schurSolve's A block is applyA (linsolve.cpp:644)
    # One lockstep batch for all p + nM inner columns (schurSolve batches by
    # the context's max_nrhs).
    nm = ToeplitzMatvec(rep, max_nrhs=1).sizeM()
    ops = ToeplitzMatvec(rep, max_nrhs=args.schur_batch or (cfg.nrhs + nm))
    V = np.zeros((ops.size(), cfg.nrhs), complex)
    V[:cfg.n] = gen.rhs_normal(cfg.n, cfg.nrhs, 4)
    sopt = SolverOptions(tol=cfg.tol, maxIter=cfg.max_iter, restart=cfg.restart)
    ops.schur_solve(V, sopt)
    t0 = time.perf_counter()
    g = ops.schur_solve(V, sopt)
    out["schur_ms"] = 1e3 * (time.perf_counter() - t0)
    out["schur_inner_columns"] = cfg.nrhs + ops.sizeM()
    out["schur_residual"] = max(g.residual)
    if not args.no_cpu:
        import oracle
        o = oracle.Oracle.from_rep(rep)
        t0 = time.perf_counter()
        r = o.schur(V, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart, nthreads=0)
        out["cpu_oracle_schur_ms_all_cores"] = 1e3 * (time.perf_counter() - t0)
        out["schur_parity_rel_err"] = float(np.linalg.norm(g.current - r["x"]) / np.linalg.norm(r["x"]))
print(json.dumps(out))
