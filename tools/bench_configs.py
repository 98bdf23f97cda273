"""Every BASELINE config on one GPU (the bench.py line covers C2 only):
device-resident operator applications (back-to-back, CUDA events), the
kernel-bound roofline of each, GMRES time per inner iteration over a fixed
budget (C1 to convergence), and the oracle's CPU time on a bounded sample.

    python tools/bench_configs.py [--configs C1,C2,C3,C4,C5] [--out file.json]

Rooflines: single-RHS configs are HBM-bound; the bytes are what one apply
must move (half spectrum once, xhat / yhat, x / y, as in bench.py) against
MEASURED_PEAKS.json hbm_gbs. G48 / G40 are shapes outside the persistent
kernel's instantiations (the multi-launch apply.cu chain). C3's
162-column apply is FP64-bound: 8 m^2 nrhs bins flops against the DMMA peak
measured by tools/fp64test.cu (37.1 TF/s)."""
import argparse
import json
import os
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, Config, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen, rhs_for  # noqa: E402

# Shapes outside the persistent kernel's instantiations (matvec_persistent.cu):
# the multi-launch apply.cu chain, measured on the same byte count.
EXTRA = {
    "G48": Config("G48", 48, 48, 96, 1, 8, 5, "normal", 50),   # 128x128 bins, m = 96
    "G40": Config("G40", 40, 24, 64, 1, 8, 6, "normal", 50),   # 64x128 bins, m = 64
}
from paper_2506_04710_b200._lib import TBT_DEVICE  # noqa: E402

DMMA_TFLOPS = 37.1  # tools/fp64test.cu, mma.sync.m8n8k4.f64 on this B200 pool


def hbm_peak():
    try:
        return float(json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, n, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / n


def apply_bytes(cfg, info):
    """Algorithmic bytes of one apply (SURVEY.md 8(d) with the stored half
    spectrum): spectrum once, xhat read + yhat written, x read + y written.
    Transform intermediates are not counted (bench.py uses the same)."""
    c16 = 16
    spectrum = info.pairs * cfg.m * cfg.m * c16
    vec = 2 * info.bins * cfg.m * c16 * cfg.nrhs
    return spectrum + vec + 2 * cfg.n * c16 * cfg.nrhs


def cpu_apply(rep, cfg, seconds, cols=1):
    """CPU matvecs/s on `cols` host threads (one column each): the reference's
    own applyA (oracle/_ref/libref_linsolve.so, kind "reference") up to C3,
    the oracle port beyond (the reference builds its spectra on one thread).
    Returns the oracle too (for the GMRES timing)."""
    import tempfile

    import oracle
    import bench
    t0 = time.perf_counter()
    o = oracle.Oracle.from_rep(rep, precompute=True, nthreads=0)
    ref = None
    if cfg.n * cfg.m <= 4_000_000:
        with tempfile.TemporaryDirectory() as td:
            ref = bench.reference_operator(cfg, td)
    pre = time.perf_counter() - t0
    X = np.asfortranarray(gen.rhs_normal(cfg.n, cols, 77))
    fn = (lambda: ref.apply_a_cols(X, threads=cols)) if ref is not None else (lambda: o.apply_cols(X, nthreads=cols))
    fn()
    cnt, t0 = 0, time.perf_counter()
    while True:
        fn()
        cnt += cols
        el = time.perf_counter() - t0
        if el >= seconds and cnt >= 2 * cols:
            break
    return o, {"matvecs_per_s": cnt / el, "threads": cols, "sample": f"{cnt} matvecs in {el:.1f} s",
               "kind": "reference" if ref is not None else "port", "spectra_precompute_s": pre}


def run(name, args, out):
    cfg = CONFIGS[name] if name in CONFIGS else EXTRA[name]
    res = {"config": name, "shape": f"{cfg.nx}x{cfg.ny}, m={cfg.m}, nrhs={cfg.nrhs}"}
    rep = ToeplitzRep.synthetic(cfg)
    stream = torch.cuda.Stream()
    embeds = ["pow2", "smooth"] if name == "C3" else ["pow2"]
    for embed in embeds:
        op = ToeplitzMatvec(rep, max_nrhs=cfg.nrhs, embed=embed)
        op.set_stream(stream.cuda_stream)
        info = op.info()
        K = cfg.nrhs
        x = torch.from_numpy(np.ascontiguousarray(gen.rhs_normal(cfg.n, K, 3).T)).cuda()
        y = torch.empty_like(x)
        with torch.cuda.stream(stream):
            f = lambda: op.apply_device(x.data_ptr(), y.data_ptr(), K)  # noqa: E731
            for _ in range(3):
                f()
            n = max(3, min(2000, int(0.5 / max(1e-6, timed(f, 2, stream) * 1e-3))))
            ms = timed(f, n, stream)
        r = {"embedding": f"{info.L1}x{info.L0}", "apply_path": info.apply_path, "ms_per_apply": ms,
             "column_matvecs_per_s": K / (ms * 1e-3), "applies_timed": n}
        if K == 1:
            b = apply_bytes(cfg, info)
            r["roofline"] = {"bound": "hbm", "bytes": b, "achieved_gbs": b / (ms * 1e-3) / 1e9,
                             "peak_gbs": hbm_peak(), "frac": b / (ms * 1e-3) / 1e9 / hbm_peak()}
        else:
            fl = 8.0 * cfg.m * cfg.m * K * info.bins
            r["roofline"] = {"bound": "fp64 tensor (DMMA)", "flops": fl, "achieved_tflops": fl / (ms * 1e-3) / 1e12,
                             "peak_tflops": DMMA_TFLOPS, "frac": fl / (ms * 1e-3) / 1e12 / DMMA_TFLOPS}
        # GMRES: device-resident b / x, second solve (workspace and graph cached)
        B = np.asarray(rhs_for(cfg)).reshape(cfg.n, -1)
        bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
        xd = torch.empty_like(bd)
        budget = {"C1": cfg.max_iter, "C2": 200, "C3": 50, "C4": 100, "C5": 10}.get(name, 50)
        opt = SolverOptions(tol=cfg.tol, maxIter=budget, restart=cfg.restart)
        for rep_i in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g = op.gmres(None, opt, raise_on_fail=False, where=TBT_DEVICE, b_ptr=bd.data_ptr(),
                         x_ptr=xd.data_ptr(), nrhs=K, hist_cap=4 * budget + 8)
            e1.record(stream)
            e1.synchronize()
        gms = e0.elapsed_time(e1)
        its = max(g.iterations)
        r["gmres"] = {"iteration_budget": budget, "restart": cfg.restart, "iterations": its,
                      "converged_columns": int(sum(g.converged)), "ms_total": gms,
                      "ms_per_iteration": gms / max(its, 1), "max_final_residual": float(max(g.residual))}
        res[embed] = r
        del op
        torch.cuda.empty_cache()
    if name in EXTRA:
        pass
    elif name != "C5" and not args.no_cpu:
        cols = min(os.cpu_count() or 1, cfg.nrhs)
        o, cpu = cpu_apply(rep, cfg, seconds={"C1": 3, "C2": 8, "C3": 10, "C4": 10}[name], cols=cols)
        if name in ("C1", "C2"):
            b = np.asarray(rhs_for(cfg)).reshape(cfg.n, -1)[:, 0]
            t0 = time.perf_counter()
            it = {"C1": cfg.max_iter, "C2": 20}[name]
            rr = o.gmres(b, tol=cfg.tol, max_iter=it, restart=cfg.restart)
            el = time.perf_counter() - t0
            cpu["gmres_ms_per_iteration"] = 1e3 * el / max(rr["iterations"][0], 1)
            cpu["gmres_sample"] = f"{rr['iterations'][0]} iterations, 1 thread"
        res["cpu_oracle"] = cpu
    elif name == "C5":
        res["cpu_oracle"] = "not run: the oracle needs ~58 GB of host RAM for C5 (SURVEY.md 8(d))"
    out.append(res)
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    out = []
    for name in args.configs.split(","):
        run(name, args, out)
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
