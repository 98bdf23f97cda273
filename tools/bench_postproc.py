"""Row f4 measurement on the C3 shape (18 x 9 array, m = 128, 162 ports):
port network and embedded element patterns, device vs oracle (one core)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, array_farfield, port_network  # noqa: E402
from test_postproc import synth  # noqa: E402

cfg = CONFIGS["C3"]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg))
ndir = int(sys.argv[1]) if len(sys.argv) > 1 else 362
e = [0, 0, 0, 0, cfg.m, 0, 0, 0, 0]
tensors, d, cur, n = synth(cfg.nx, cfg.ny, e, ndir, 162)
rng = np.random.default_rng(0)
feed = np.arange(162) * cfg.m + rng.integers(0, cfg.m, 162)
z0 = np.full(162, 50.0)
out = {"config": "C3 shape", "ports": 162, "directions": ndir}


def best(fn, n=3):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), r


t, g = best(lambda: port_network(op, cur, feed, 0.02, z0))
out["port_network_gpu_ms"] = 1e3 * t
t, r = best(lambda: oracle.port_network(cur, feed, 0.02, z0), 1)
out["port_network_oracle_ms"] = 1e3 * t
out["port_network_rel_err_s"] = float(np.linalg.norm(g["s"] - r["s"]) / np.linalg.norm(r["s"]))
W = np.eye(162)
t, (co, cx) = best(lambda: array_farfield(op, tensors, e, d, 0.5, 0.5, 2.0, 376.73, cur, W))
out["element_patterns_gpu_ms"] = 1e3 * t
t, (rco, rcx) = best(lambda: oracle.array_farfield(cfg.nx, cfg.ny, e, tensors, d, 0.5, 0.5, 2.0, 376.73, cur, W), 1)
out["element_patterns_oracle_ms"] = 1e3 * t
out["element_patterns_rel_err"] = float(np.linalg.norm(co - rco) / np.linalg.norm(rco))
print(json.dumps(out))
