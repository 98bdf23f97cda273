"""Short C2 GMRES run for ncu launch lists (fixed iteration budget)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, rhs_for  # noqa: E402
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rep = ToeplitzRep.synthetic(cfg)
op = ToeplitzMatvec(rep, max_nrhs=cfg.nrhs, embed=sys.argv[3] if len(sys.argv) > 3 else "pow2")
b = np.asarray(rhs_for(cfg))
r = op.gmres(b, SolverOptions(tol=cfg.tol, maxIter=iters, restart=cfg.restart), raise_on_fail=False)
print("ok", r.iterations, r.residual)
