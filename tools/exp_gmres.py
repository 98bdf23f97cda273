"""GMRES time per inner iteration (device events around a fixed-budget
solve, second solve of the context) under the current environment knobs.

    TBT_GMRES=graph python tools/exp_gmres.py --config C2 --iters 200
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, rhs_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--tag", default="")
args = ap.parse_args()
cfg = CONFIGS[args.config]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
st = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
b = np.asarray(rhs_for(cfg))
o = SolverOptions(tol=cfg.tol, maxIter=args.iters, restart=cfg.restart)
best = None
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = op.gmres(b, o, raise_on_fail=False)
    e1.record(st)
    st.synchronize()
    ms = e0.elapsed_time(e1)
    best = ms if best is None else min(best, ms)
it = r.iterations[0]
print(f"{args.tag:16s} {args.config} GMRES {it} its: {best:.3f} ms, {1e3 * best / it:.2f} us/iteration, "
      f"residual {r.residual[0]:.6e}", flush=True)
