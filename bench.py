#!/usr/bin/env python3
"""Benchmark: block-Toeplitz matvecs/s (+ GMRES time per iteration) on
BASELINE.json's config 2 (32x32 array, m = 64, complex128, 1 RHS).

One step = one application of the operator (K2 forward FFT passes -> K3
bin-pair product -> K4 inverse passes -> edge/corner correction) to a
device-resident vector. The headline `value` times K back-to-back steps
between two CUDA events on the launching stream: the dominant input, the
134 MB half spectrum, is larger than the 126 MB L2, so every step reads it
from HBM; `cold_l2_ms_per_step` repeats the step with an untimed 256 MiB L2
flush before each one.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--impl reference times the reference ITSELF on the host CPU: its own
applyA (proj/src/linsolve.cpp:260-290) compiled unchanged into
oracle/_ref/libref_linsolve.so (oracle/Makefile, against a functional
Eigen-subset shim), every host thread, one column per thread as the
reference's parallelFor does (linsolve.cpp:572). That process never maps
libtbt.so: its inputs come from oracle/liboracle.so's copy of the seeded
generator (csrc/gen.cpp), and it checks /proc/self/maps before timing.

N > 1 (torchrun): the headline is C2 through the bin-sharded operator over
all N GPUs (csrc/dist.cu: bins split by level-0 column groups, row slabs,
NCCL all-to-all transposes, one-row halo exchange for the correction), so
total work is fixed and scaling is "strong"; device time per matvec is the
max over ranks, and the exposed all-to-all time is reported beside it. The
independent-replica numbers (one frequency point per GPU) stay in
"replicas".

"sharded" (every N, --no-sharded skips it): C4 through the same multi-GPU
operator — device ms per matvec and exposed NCCL ms per matvec (max over
ranks; at N = 1 a one-rank communicator, i.e. the sharded path's own
overhead).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

CONFIG = "C2"
L2_FLUSH_BYTES = 256 << 20


def l2_flush(buf, k):
    """Untimed L2 flush between steps: write a buffer twice the L2 size,
    then read it back, so the flush's own dirty lines are written back
    before the next timed step starts (a write-only flush would leave
    ~126 MB of dirty lines for the timed kernels to evict)."""
    buf.fill_(float(k))
    return buf.sum()


def measured_hbm():
    p = REPO / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"


TRAFFIC_FILES = ("r2d_traffic.json", "r2c_traffic.json", "r2b_traffic.json", "r2_traffic.json", "r1_traffic.json")  # newest capture first


def ncu_traffic(key):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (the newest of profiles/r2d, r2c, r2b, r2, r1 _traffic.json), and the file it came from."""
    for name in TRAFFIC_FILES:
        try:
            return json.loads((REPO / "profiles" / name).read_text())[key]["dram_bytes_per_launch"], name
        except Exception:
            continue
    return None, None


def workload_desc(cfg):
    L0 = 1 << (2 * cfg.nx - 1 - 1).bit_length()
    L1 = 1 << (2 * cfg.ny - 1 - 1).bit_length()
    return (f"{cfg.name}: {cfg.nx}x{cfg.ny} array, m={cfg.m}, {cfg.nrhs} RHS, complex128, "
            f"pow2 circulant embedding {L1}x{L0}, diag+rank-{cfg.rank} edge/corner corrections")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during measurement."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def host_cpu():
    """Host CPU model and logical core count (record them)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def reference_operator(cfg, tmpdir):
    """The reference's own ToeplitzMatvec (oracle/_ref/libref_linsolve.so)
    on cfg's generator blocks, read from a ZTOE1 cache by its own
    loadBlockCache (untimed, one-time). None when the library is absent."""
    import oracle
    if oracle.ref_linsolve() is None:
        return None
    from paper_2506_04710_b200 import gen
    path = os.path.join(tmpdir, f"{cfg.name}.ztoe1")
    oracle.write_ztoe1_a(path, cfg.nx, cfg.ny, cfg.m, gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed))
    op = oracle.RefOperator(path)
    os.unlink(path)
    return op


def cpu_sample(rep, cfg, seconds=12.0, threads=1, prefer_reference=True):
    """The reference's applyA timed on host cores (kind "reference"), or the
    oracle port (kind "port") when oracle/_ref is absent or not preferred
    (C4: the reference builds its 4.3 GB of spectra on one thread, ~1 min):
    returns (matvec/s, count, elapsed, precompute s, kind, what)."""
    import tempfile

    import numpy as np

    import oracle
    from paper_2506_04710_b200 import gen
    X = np.asfortranarray(gen.rhs_normal(cfg.n, threads, 77))
    t0 = time.perf_counter()
    ref = None
    if prefer_reference:
        with tempfile.TemporaryDirectory() as td:
            ref = reference_operator(cfg, td)
    if ref is not None:
        fn = lambda: ref.apply_a_cols(X, threads=threads)  # noqa: E731
        kind, what = "reference", "the reference's own applyA (oracle/_ref/libref_linsolve.so, linsolve.cpp:260-290)"
    else:
        o = oracle.Oracle.from_rep(rep, precompute=True, nthreads=0)
        fn = lambda: o.apply_cols(X, nthreads=threads)  # noqa: E731
        kind, what = "port", "oracle/oracle.cpp restatement of applyA + correction"
    t_pre = time.perf_counter() - t0  # spectra precompute: one-time, untimed
    fn()  # warm
    count, t0 = 0, time.perf_counter()
    while True:
        fn()
        count += threads
        el = time.perf_counter() - t0
        if el >= seconds and count >= 3:
            break
    return count / el, count, el, t_pre, kind, what


def cpu_sample_c5(seconds_cap=60.0):
    """C5 on the host CPU: the reference algorithm's applyA does not fit
    host memory there (38.65 GB of spectra + 19.2 GB of generators), so the
    oracle times a bounded sample (orc_sampled_apply): all 192 forward 2-D
    FFTs of x plus the per-row work (products over every bin and source
    function, inverse 2-D FFT, crop) of 4 of the 192 output rows, one
    thread; the matvec time is t_fwd + 192/4 * t_rows."""
    import numpy as np

    import oracle
    from paper_2506_04710_b200 import CONFIGS, gen
    cfg = CONFIGS["C5"]
    rows = [3, 61, 130, 191]
    x = gen.rhs_normal(cfg.n, 1, 77)[:, 0]
    t0 = time.perf_counter()
    _, tf, tr = oracle.sampled_apply(cfg.nx, cfg.ny, cfg.m, cfg.seed, rows, x)
    est = tf + cfg.m / len(rows) * tr
    return {"value": 1.0 / est, "unit": "matvec/s", "cores": 1, "kind": "port",
            "sample": f"C5 applyA restated (oracle/oracle.cpp orc_sampled_apply, linsolve.cpp:260-290): all "
                      f"{cfg.m} forward 2-D FFTs ({tf:.2f} s) + {len(rows)} of {cfg.m} output rows "
                      f"({tr:.3f} s), one thread; matvec = t_fwd + {cfg.m}/{len(rows)} t_rows = {est:.2f} s; "
                      f"the reference itself needs ~58 GB host RAM at C5",
            "wall_s": time.perf_counter() - t0}


def run_reference(args):
    """--impl reference: the reference itself on the host CPU."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import tempfile

    import numpy as np

    import oracle
    oracle.bind_inputs()  # inputs from liboracle's copy of csrc/gen.cpp
    from paper_2506_04710_b200 import CONFIGS, gen
    cfg = CONFIGS[CONFIG]
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as td:
        ref = reference_operator(cfg, td)
    if ref is not None:
        fn = lambda X: ref.apply_a_cols(X, threads=cores)  # noqa: E731
        kind = "reference"
        what = "the reference's own applyA (oracle/_ref/libref_linsolve.so: proj/src/linsolve.cpp compiled unchanged)"
    else:
        from paper_2506_04710_b200 import ToeplitzRep
        o = oracle.Oracle.from_rep(ToeplitzRep.synthetic(cfg), precompute=True, nthreads=0)
        fn = lambda X: o.apply_cols(X, nthreads=cores)  # noqa: E731
        kind, what = "port", "oracle/oracle.cpp restatement of applyA + correction"
    assert not oracle.product_mapped(), "reference arm must not map libtbt.so"
    X = np.asfortranarray(gen.rhs_normal(cfg.n, cores, 5))
    for _ in range(max(1, min(args.warmup, 3))):
        fn(X)
    # Each step: one batch of `cores` independent matvecs (one column per thread);
    # steps are bounded so the whole run stays within a few minutes.
    steps = max(1, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(steps):
        fn(X)
    el = time.perf_counter() - t0
    value = steps * cores / el
    sample = f"{steps} steps x {cores} concurrent {cfg.name} matvecs ({what}), one column per thread as parallelFor"
    line = {
        "impl": "reference", "metric": f"block-Toeplitz matvecs/s ({cfg.name}, complex128)", "value": value,
        "unit": "matvec/s", "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded generator, include/tbt_gen.h)",
        "config": {"workload": workload_desc(cfg), "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": cores, "kind": kind, "sample": sample,
                         "host": host_cpu()},
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_mapped": oracle.product_mapped(),
        "note": "the reference has no GPU path; the BASELINE edge/corner correction is not a reference feature "
                "and is not in this arm (<0.5% of the CPU work)",
    }
    emit(line)
    return 0


def large_configs(local, with_cpu):
    """C4 (64x64, m=128) and C5 (128x128, m=192) on this GPU, as extra keys
    of the bench line so the driver observes them: device-resident applies
    (back-to-back, CUDA events on the context stream; both spectra exceed
    L2 by 34x / 160x), the roofline on the same algorithmic bytes as the
    headline, GMRES(50) time per inner iteration over a fixed budget
    (second solve: workspace and graphs cached), and a bounded CPU sample."""
    import numpy as np
    import torch

    from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen, rhs_for
    from paper_2506_04710_b200._lib import TBT_DEVICE
    peak, _ = measured_hbm()
    dev = f"cuda:{local}"
    out = {}
    for name, n_apply, budget in (("C4", 200, 50), ("C5", 30, 50)):
        cfg = CONFIGS[name]
        t0 = time.perf_counter()
        rep = ToeplitzRep.synthetic(cfg)
        op = ToeplitzMatvec(rep, max_nrhs=1, device=local)
        setup_s = time.perf_counter() - t0
        try:
            st = torch.cuda.Stream(device=dev)
            op.set_stream(st.cuda_stream)
            info = op.info()
            x = torch.from_numpy(np.ascontiguousarray(gen.rhs_normal(cfg.n, 1, 3)[:, 0])).to(dev)
            y = torch.empty_like(x)
            for _ in range(3):
                op.apply_device(x.data_ptr(), y.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(n_apply):
                op.apply_device(x.data_ptr(), y.data_ptr())
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / n_apply
            kbytes = 16 * (info.pairs * cfg.m * cfg.m + 2 * info.bins * cfg.m + 2 * cfg.n)
            b = torch.from_numpy(np.ascontiguousarray(np.asarray(rhs_for(cfg)).reshape(cfg.n))).to(dev)
            xd = torch.empty_like(b)
            opt = SolverOptions(tol=cfg.tol, maxIter=budget, restart=cfg.restart)
            for _ in range(2):
                e0.record(st)
                g = op.gmres(None, opt, raise_on_fail=False, where=TBT_DEVICE, b_ptr=b.data_ptr(),
                             x_ptr=xd.data_ptr(), nrhs=1, hist_cap=4 * budget + 8)
                e1.record(st)
                e1.synchronize()
            gms = e0.elapsed_time(e1)
            out[name] = {
                "workload": workload_desc(cfg), "ms_per_apply": ms, "matvec_per_s": 1e3 / ms, "applies_timed": n_apply,
                "roofline": {"bound": "hbm", "bytes_per_launch": kbytes, "achieved": kbytes / (ms * 1e-3) / 1e9,
                             "peak": peak, "unit": "GB/s", "frac": kbytes / (ms * 1e-3) / 1e9 / peak},
                "kernels_per_apply": info.kernels_per_apply, "apply_path": info.apply_path,
                "gmres": {"restart": cfg.restart, "iteration_budget": budget, "iterations": g.iterations[0],
                          "matvecs": g.matvecs, "ms_total": gms, "ms_per_iteration": gms / max(g.iterations[0], 1),
                          "final_true_residual": g.residual[0]},
                "setup_s": setup_s}
        finally:
            op.close()
            del rep
            torch.cuda.empty_cache()
        if with_cpu and name == "C4":
            v, cnt, el, t_pre, kind, what = cpu_sample(ToeplitzRep.synthetic(cfg), cfg, seconds=8.0, threads=1,
                                                       prefer_reference=False)
            out[name]["cpu_baseline"] = {"value": v, "unit": "matvec/s", "cores": 1, "kind": kind,
                                         "sample": f"{cnt} single-thread matvecs in {el:.1f} s ({what}); spectra "
                                                   f"precompute {t_pre:.1f} s excluded"}
        if with_cpu and name == "C5":
            out[name]["cpu_baseline"] = cpu_sample_c5()
    return out


SHARDED_TIMEOUT_S = 240


def sharded_measure(name, world, rank, local, dist, steps=30, warmup=3, gmres_iters=20, e2e_steps=0):
    """Config `name` through the multi-GPU operator (csrc/dist.cu): bins split
    by level-0 column groups, element-row slabs, NCCL all-to-all transposes
    around the column transforms, one-row halo exchange for the correction.
    Device time per matvec (CUDA events on the context stream, max over
    ranks), the exposed NCCL time per matvec (events around each exchange,
    tbt_set_timing), GMRES time per iteration over a fixed budget, and
    (e2e_steps > 0) matvecs/s through tbt_apply with this rank's pinned host
    slab copied in and out every call (max over ranks)."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2506_04710_b200 import (CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, dist_unique_id, gen,
                                       init_from_torch)
    from paper_2506_04710_b200._lib import TBT_DEVICE, TBT_HOST, lib
    cfg = CONFIGS[name]
    d = init_from_torch() if dist is not None else (1, 0, dist_unique_id())
    op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1, device=local, dist=d)
    try:
        st = torch.cuda.Stream()
        op.set_stream(st.cuda_stream)
        r0, r1 = op.rows()
        dev = f"cuda:{local}"
        xs = np.ascontiguousarray(gen.rhs_normal(cfg.n, 1, 1000)[r0 * cfg.nx * cfg.m:r1 * cfg.nx * cfg.m, 0])
        x = torch.from_numpy(xs).to(dev)
        y = torch.empty_like(x)
        for _ in range(warmup):
            op.apply_device(x.data_ptr(), y.data_ptr())
        st.synchronize()
        if dist is not None:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            op.apply_device(x.data_ptr(), y.data_ptr())
        e1.record(st)
        st.synchronize()
        ms = e0.elapsed_time(e1) / steps
        op.set_timing(True)
        for _ in range(steps):
            op.apply_device(x.data_ptr(), y.data_ptr())
        comm_total, cnt = op.timing_read()
        op.set_timing(False)
        comm = comm_total / steps
        e2e_s = None
        if e2e_steps > 0:
            xh = torch.from_numpy(xs.copy()).pin_memory()
            yh = torch.empty_like(xh).pin_memory()
            for _ in range(warmup):
                lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                if lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST):
                    raise RuntimeError("tbt_apply failed")
            e2e_s = time.perf_counter() - t0
        # Distributed GMRES(restart) over a fixed budget (column-blocked
        # Arnoldi, two all-reduces per iteration), b / x device-resident slabs.
        opt = SolverOptions(tol=cfg.tol, maxIter=gmres_iters, restart=cfg.restart)
        xd = torch.empty_like(x)

        def solve(o):
            return op.gmres(None, o, raise_on_fail=False, where=TBT_DEVICE, b_ptr=x.data_ptr(), x_ptr=xd.data_ptr(),
                            nrhs=1)

        solve(SolverOptions(tol=cfg.tol, maxIter=2, restart=cfg.restart))
        if dist is not None:
            dist.barrier()
        e0.record(st)
        res = solve(opt)
        e1.record(st)
        e1.synchronize()
        gms = e0.elapsed_time(e1) / max(res.iterations[0], 1)
        vals = [ms, comm, gms, e2e_s if e2e_s is not None else 0.0]
        if dist is not None:
            t = torch.tensor(vals, device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            vals = [float(v) for v in t.tolist()]
        ms, comm, gms, e2e_s = vals
        info = op.info()
        out = {"config": f"{workload_desc(cfg)}; sharded over the job's {world} GPU(s)", "n_gpus": world,
               "ms_per_matvec": ms, "matvec_per_s": 1e3 / ms, "exposed_nccl_ms_per_matvec": comm,
               "nccl_sections_per_matvec": cnt / steps, "gmres_ms_per_iteration": gms,
               "gmres_iterations": res.iterations[0], "element_rows_this_rank": [r0, r1],
               "spectrum_pairs_this_rank": info.pairs,
               "timing": "CUDA events on the context stream, max over ranks"}
        if e2e_steps > 0:
            out["e2e_matvec_per_s"] = e2e_steps / e2e_s
            out["e2e_bytes_per_rank"] = 2 * xs.nbytes
        return out
    finally:
        op.close()


_JSON_FD = None


def _quiet_stdout():
    """Points fd 1 at stderr for the rest of the run and keeps the real
    stdout for the one JSON line: native libraries print to stdout (NCCL's
    version banner on communicator init), which must not precede the line."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    """Writes the bench's single JSON line to the real stdout."""
    sys.stdout.flush()
    try:
        import ctypes
        ctypes.CDLL(None).fflush(None)  # C stdio buffers of native libraries
    except OSError:
        pass
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    _quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--gmres-iters", type=int, default=200)
    ap.add_argument("--no-sharded", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the C4 / C5 extra keys")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen, rhs_for
    from paper_2506_04710_b200._lib import TBT_DEVICE

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = CONFIGS[CONFIG]
    rep = ToeplitzRep.synthetic(cfg)
    op = ToeplitzMatvec(rep, max_nrhs=1, device=local)
    stream = torch.cuda.Stream()
    op.set_stream(stream.cuda_stream)
    info = op.info()

    x_host = np.asarray(gen.rhs_normal(cfg.n, 1, 1000 + rank)[:, 0])
    x = torch.from_numpy(x_host.copy()).to(f"cuda:{local}")
    y = torch.empty_like(x)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=f"cuda:{local}")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    K, W = args.steps, args.warmup
    with torch.cuda.stream(stream):
        for _ in range(W):
            op.apply_device(x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    with clocks:
        # ---- value: K back-to-back device-resident applies (the GMRES usage
        # pattern). The dominant input, the half spectrum (134 MB at C2), is
        # larger than L2 (126 MB) and is streamed with an evict-first policy,
        # so every step reads it from HBM.
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for k in range(K):
                op.apply_device(x.data_ptr(), y.data_ptr())
            e1.record(stream)
        stream.synchronize()
        barrier()
        total_ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        value = world * K / (total_ms / 1e3)

        # ---- cold-L2 step time (reported beside): L2 flushed between steps
        kc = min(K, 200)
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(kc)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(kc)]
        with torch.cuda.stream(stream):
            for k in range(kc):
                l2_flush(flush, k)
                ev0[k].record(stream)
                op.apply_device(x.data_ptr(), y.data_ptr())
                ev1[k].record(stream)
        stream.synchronize()
        cold_ms = statistics.median(a.elapsed_time(b) for a, b in zip(ev0, ev1))

        # ---- roofline of the dominant kernel
        if info.apply_path == 2:
            # One persistent kernel per apply: its launch IS the timed step.
            # Phase split from %globaltimer stamps of a few extra applies.
            op.phase_times(True)
            phases = []
            with torch.cuda.stream(stream):
                for k in range(min(K, 50)):
                    l2_flush(flush, k)
                    op.apply_device(x.data_ptr(), y.data_ptr())
                    stream.synchronize()
                    phases.append(op.phase_times(True))
            op.phase_times(False)
            phase_us = [statistics.median(p[i] for p in phases) for i in range(5)]
            k3_ms = None
        else:
            op.set_timing(True)
            with torch.cuda.stream(stream):
                for k in range(K):
                    l2_flush(flush, k)
                    op.apply_device(x.data_ptr(), y.data_ptr())
            k3_total, k3_count = op.timing_read()
            op.set_timing(False)
            k3_ms = k3_total / max(k3_count, 1)
            phase_us = None

        # ---- e2e: C-ABI call with pinned HOST buffers (H2D + apply + D2H + sync per step)
        xh = torch.from_numpy(x_host.copy()).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        import ctypes as C
        from paper_2506_04710_b200._lib import TBT_HOST, lib
        for _ in range(W):
            lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
        barrier()
        ke = max(10, K // 2)
        t0 = time.perf_counter()
        for _ in range(ke):
            st = lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
            assert st == 0
        e2e_single_s = time.perf_counter() - t0
        # Streamed: tbt_apply_many over batches of distinct pinned host
        # vectors; every vector's H2D copy, apply and D2H copy is inside the
        # timed region, consecutive vectors overlap on the copy engines.
        nb = 64
        xs_many = torch.from_numpy(np.ascontiguousarray(gen.rhs_normal(cfg.n, nb, 77).T)).pin_memory()
        ys_many = torch.empty_like(xs_many).pin_memory()
        op.apply_many_ptr(xs_many.data_ptr(), ys_many.data_ptr(), nb)  # warm-up (slot allocation)
        ref_y = ys_many[3].numpy().copy()
        barrier()
        calls = max(1, ke // nb)
        t0 = time.perf_counter()
        for _ in range(calls):
            op.apply_many_ptr(xs_many.data_ptr(), ys_many.data_ptr(), nb)
        e2e_s = time.perf_counter() - t0
        assert np.array_equal(ys_many[3].numpy(), ref_y)  # same vector, same bits every call
        if dist is not None:
            t = torch.tensor([e2e_s, e2e_single_s], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s, e2e_single_s = (float(v) for v in t.tolist())
        e2e = world * calls * nb / e2e_s
        e2e_single = world * ke / e2e_single_s

        # ---- GMRES: fixed budget (C2 stalls under GMRES(50)+Jacobi)
        gm = None
        if not args.no_gmres:
            b = np.asarray(rhs_for(cfg))
            bd = torch.from_numpy(b.copy()).to(f"cuda:{local}")
            xd = torch.empty_like(bd)
            opt = SolverOptions(tol=cfg.tol, maxIter=args.gmres_iters, restart=cfg.restart)
            hc = 4 * args.gmres_iters

            def solve():
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                res = op.gmres(None, opt, raise_on_fail=False, where=TBT_DEVICE, b_ptr=bd.data_ptr(),
                               x_ptr=xd.data_ptr(), nrhs=1, hist_cap=hc)
                g1.record(stream)
                g1.synchronize()
                return res, g0.elapsed_time(g1)

            barrier()
            _, first_ms = solve()  # includes workspace allocation + inner-loop graph instantiation
            res, gms = solve()     # cached workspace / graph (repeated solves, e.g. a frequency sweep)
            gm = {"config": cfg.name, "restart": cfg.restart, "iterations": res.iterations[0],
                  "matvecs": res.matvecs, "ms_total": gms, "ms_per_iteration": gms / max(res.iterations[0], 1),
                  "first_solve_ms_total": first_ms, "orthogonalisation": "low-synchronisation MGS",
                  "final_true_residual": res.residual[0], "converged": bool(res.converged[0]),
                  "note": "fixed budget: the BASELINE generator stalls under GMRES(50)+Jacobi (SURVEY.md App. B)"}

    peak, peak_src = measured_hbm()
    c16 = 16
    mm = cfg.m * cfg.m * c16
    spectrum = info.pairs * mm                       # half spectrum, read once
    vec_k3 = 2 * info.bins * cfg.m * c16             # xhat read + yhat write by the bin products
    step_mean = total_ms / K
    # Algorithmic bytes per launch (with the half spectrum this
    # design stores): the stored spectrum read once, xhat read + yhat written
    # by the bin products, x read + y written once. Transform intermediates
    # (the row-transformed grid T, xhat written by the forward pass, yhat read
    # by the inverse) live in L2 and are NOT counted; ncu's DRAM bytes per
    # launch are reported beside as `traffic`.
    kbytes = spectrum + vec_k3 + 2 * cfg.n * c16
    if info.apply_path == 2:
        kms = step_mean
        kname = "matvec_persistent (K2+K3+K4 phases in one persistent kernel, 1 launch per step)"
    else:
        kms = k3_ms
        kname = "binprod (K3, bin-pair product)"
    achieved = kbytes / (kms * 1e-3) / 1e9
    b_alg_full = 16 * (info.bins * cfg.m * cfg.m + (2 * cfg.m * info.bins + 2 * cfg.n))
    traffic, tsrc = ncu_traffic(f"{cfg.name}_matvec_persistent") if info.apply_path == 2 else (None, None)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": f"profiles/{tsrc} (ncu --set full, one launch)" if tsrc else None,
            "kernel": kname, "bytes_per_launch": kbytes,
            "bytes_definition": "half spectrum (npairs*m^2*16) + xhat/yhat (2*L*m*16) + x/y (2*n*16)",
            "ms_per_launch": kms, "peak_source": peak_src}
    if phase_us is not None:
        roof["phase_us"] = dict(zip(["rows+corr", "cols", "binprod", "inv_cols", "inv_rows"], phase_us))
        if phase_us[2] > 0:
            roof["binprod_phase_gbs"] = (spectrum + vec_k3) / (phase_us[2] * 1e-6) / 1e9
            roof["k3_phase_frac"] = roof["binprod_phase_gbs"] / peak

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cnt, el, t_pre, kind, what = cpu_sample(rep, cfg, seconds=12.0, threads=1)
        cpu = {"value": v, "unit": "matvec/s", "cores": 1, "kind": kind, "host": host_cpu(),
               "sample": f"{cnt} single-thread {cfg.name} matvecs in {el:.1f} s ({what}; -O3, applyA is serial in "
                         f"the reference); one-time spectra precompute {t_pre:.2f} s excluded"}

    line = {
        "metric": f"block-Toeplitz matvecs/s ({cfg.name}, complex128)",
        "value": value, "unit": "matvec/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": step_mean, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded generator, include/tbt_gen.h; paper geometries unavailable)",
        "config": {"workload": workload_desc(cfg),
                   "l2": "inputs larger than L2: 134 MB half spectrum (> 126 MB L2) streamed evict-first every "
                         "step; back-to-back applies (cold_l2_ms_per_step: same apply with a 256 MiB "
                         "write + read-back L2 flush between steps)",
                   "parallelism": "replicas" if world > 1 else "single GPU",
                   "spectrum_storage": f"half (bin pairs): {info.pairs} blocks of {info.bins} bins"},
        "roofline": roof,
        "equivalent_full_spectrum_gbs": b_alg_full / (step_mean * 1e-3) / 1e9,
        "cold_l2_ms_per_step": cold_ms,
        "e2e": {"value": e2e, "unit": "matvec/s", "h2d_bytes_per_step": cfg.n * 16, "d2h_bytes_per_step": cfg.n * 16,
                "mode": "tbt_apply_many: batches of 64 distinct pinned host vectors; per vector H2D copy, apply, "
                        "D2H copy, overlapped across vectors on the copy engines; host wall clock",
                "single_call_value": e2e_single,
                "single_call_mode": "tbt_apply(TBT_HOST) per vector: zero-copy persistent kernel + stream sync"},
        "gpu_launches": K * info.kernels_per_apply,
        "clocks": clocks.summary(),
        "gmres": gm,
        "sharded": None,
        "cpu_baseline": cpu,
        "large_configs": None,
    }
    if not args.no_large and world == 1:
        try:
            line["large_configs"] = large_configs(local, rank == 0 and not args.no_cpu)
        except Exception as exc:  # reported, not fatal for the main line
            line["large_configs"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
    # ---- the bin-sharded operator on C4 across the job's
    # GPUs (a one-rank NCCL communicator at N=1): per-matvec time and the
    # exposed NCCL exchange time. A watchdog prints the line without it if a
    # collective gets stuck, so it cannot cost the main measurement.
    if not args.no_sharded:
        done = threading.Event()

        def watchdog():
            if not done.wait(SHARDED_TIMEOUT_S):
                if rank == 0:
                    line["sharded"] = {"error": f"timed out after {SHARDED_TIMEOUT_S} s"}
                    emit(line)
                os._exit(0)

        threading.Thread(target=watchdog, daemon=True).start()
        if world > 1:
            # N > 1: the headline is the bin-sharded C2 operator over all N
            # GPUs (total work fixed: strong scaling); the replica numbers
            # measured above stay in "replicas".
            try:
                sh = sharded_measure(CONFIG, world, rank, local, dist, steps=max(20, min(K, 2000)),
                                     gmres_iters=40, e2e_steps=max(10, min(K // 2, 1000)))
                line["replicas"] = {"value": line["value"], "ms_per_step": line["ms_per_step"],
                                    "e2e": line["e2e"]["value"], "scaling": "weak",
                                    "note": "N independent single-GPU replicas (frequency-sweep points)"}
                line["value"] = sh["matvec_per_s"]
                line["ms_per_step"] = sh["ms_per_matvec"]
                line["scaling"] = "strong"
                line["config"]["parallelism"] = f"bin-sharded over {world} GPUs (NCCL all-to-all transposes)"
                line["e2e"] = {"value": sh["e2e_matvec_per_s"], "unit": "matvec/s",
                               "h2d_bytes_per_step": cfg.n * 16, "d2h_bytes_per_step": cfg.n * 16,
                               "note": "each rank copies its row slab in and out per call; max over ranks"}
                line["sharded_headline"] = sh
                line["exposed_alltoall_ms_per_step"] = sh["exposed_nccl_ms_per_matvec"]
            except Exception as exc:  # the replica line stands, with the reason
                line["sharded_headline"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        try:
            line["sharded"] = sharded_measure("C4", world, rank, local, dist)
        except Exception as exc:  # reported, not fatal for the main line
            line["sharded"] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        done.set()
    if rank == 0:
        emit(line)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
