"""schurSolve on a config with margin parts, for launch lists:
    python tools/prof_schur.py [C1] [batch]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
rep = ToeplitzRep.synthetic(cfg)
rep.correction = None
rep.margin = gen.margin(cfg.nx, cfg.ny, [8, 8, 8, 8, cfg.m, 8, 8, 8, 8], cfg.seed + 7)  # as tools/bench_margin.py
nm = ToeplitzMatvec(rep, max_nrhs=1).sizeM()
batch = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.nrhs + nm
op = ToeplitzMatvec(rep, max_nrhs=batch)
V = np.zeros((op.size(), cfg.nrhs), complex)
V[:cfg.n] = gen.rhs_normal(cfg.n, cfg.nrhs, 4)
opt = SolverOptions(tol=cfg.tol, maxIter=cfg.max_iter, restart=cfg.restart)
for k in range(2):
    t0 = time.perf_counter()
    g = op.schur_solve(V, opt)
    print(f"schur {1e3 * (time.perf_counter() - t0):.1f} ms, iterations {g.iterations}, residual {max(g.residual):.2e}")
