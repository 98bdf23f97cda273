"""Per-CTA timeline of fused GMRES nodes of a restart cycle (TBT_CTATRACE=1):
the 8 trace slots hold the last 8 traced launches; they are ordered by start
time and each is shown relative to the previous node's last CTA end (event
14): first CTA start, programmatic-wait end, barriers 0..3 (last arrival /
release), C2 end, y barrier, LS dot barrier, step end (max over CTAs).

    TBT_CTATRACE=1 python tools/cta_trace_gmres.py --iters 50
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("TBT_CTATRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, rhs_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=50)
args = ap.parse_args()
cfg = CONFIGS[args.config]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
b = np.asarray(rhs_for(cfg))
o = SolverOptions(tol=cfg.tol, maxIter=args.iters, restart=cfg.restart)
op.gmres(b, o, raise_on_fail=False)
op.gmres(b, o, raise_on_fail=False)
torch.cuda.synchronize()
cnt, tr = op.cta_trace()
G = torch.cuda.get_device_properties(0).multi_processor_count
tr = tr[:, :, :G].astype(np.int64)
order = sorted(range(8), key=lambda k: tr[k][0].min())
cols = ["start", "pdl", "arr0", "rel0", "arr1", "rel1", "arr2", "rel2", "arr3", "rel3", "C2end", "ybar", "dots", "end"]
print(f"{args.config} fused GMRES nodes (us, relative to the previous node's last CTA end)")
print("     " + " ".join(f"{c:>6s}" for c in cols))
for i in range(1, 8):
    prev, cur = tr[order[i - 1]], tr[order[i]]
    t0 = prev[14].max()
    row = [cur[0].min(), cur[1].max()] + [v for kk in range(4) for v in (cur[2 + kk].max(), cur[6 + kk].max())] + \
          [cur[10].max(), cur[12].max(), cur[13].max(), cur[14].max()]
    print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:6.2f}" for x in row))
