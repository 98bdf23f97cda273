import sys; sys.path.insert(0, '/root/repo')
import numpy as np, oracle
from paper_2506_04710_b200 import Config, ToeplitzRep, ToeplitzMatvec, SolverOptions, gen
cfg = Config("t", 5, 4, 8, 1, 4, 3, "normal", 20)
rep = ToeplitzRep.synthetic(cfg)
o = oracle.Oracle.from_rep(rep)
B = gen.rhs_normal(o.n, 3, 21); B[:, 1] = 0
op = ToeplitzMatvec(rep, max_nrhs=3)
for a_only in (False, True):
    g = op.gmres(B, SolverOptions(tol=1e-9, maxIter=500, restart=12), use_a_only=a_only, raise_on_fail=False)
    r = o.gmres(B, tol=1e-9, max_iter=500, restart=12, use_a_only=a_only)
    print("a_only", a_only, g.iterations, r["iterations"], g.converged, r["converged"])
    for c in range(3):
        hg, hr = g.history[c], r["history"][c]
        n = min(len(hg), len(hr))
        print(c, len(hg), len(hr), hg[:4, 1], hr[:4, 1])
    # single column runs
    for c in (0, 2):
        op1 = ToeplitzMatvec(rep)
        g1 = op1.gmres(B[:, c].copy(), SolverOptions(tol=1e-9, maxIter=500, restart=12), use_a_only=a_only, raise_on_fail=False)
        print(" single", c, g1.iterations, g1.history[0][:4, 1])
