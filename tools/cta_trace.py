"""Per-CTA timeline of back-to-back persistent applies (TBT_CTATRACE=1):
CTA start / PDL wait / barrier arrival and release / end, relative to the
previous launch's last CTA end, with the distribution over CTAs and the
split by die (SM id < / >= half).

    TBT_CTATRACE=1 python tools/cta_trace.py --config C2
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("TBT_CTATRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--rounds", type=int, default=20)
args = ap.parse_args()
cfg = CONFIGS[args.config]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
st = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
n = op.size()
x = torch.randn(n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
G = torch.cuda.get_device_properties(0).multi_processor_count
for _ in range(20):
    op.apply_device(x.data_ptr(), y.data_ptr())
st.synchronize()
names = ["start", "pdl", "arr0", "arr1", "arr2", "arr3", "rel0", "rel1", "rel2", "rel3", "end"]
acc = {k: [] for k in names}
per_cta_b = []
gaps = []
for _ in range(args.rounds):
    for _ in range(8):
        op.apply_device(x.data_ptr(), y.data_ptr())
    cnt, tr = op.cta_trace()
    order = [(cnt - 8 + i) % 8 for i in range(8)]
    for i in range(1, 8):
        prev, cur = tr[order[i - 1]][:, :G].astype(np.int64), tr[order[i]][:, :G].astype(np.int64)
        t0 = prev[10].max()  # previous launch's last CTA end
        for k, nm in enumerate(names):
            acc[nm].append(cur[k] - t0)
        per_cta_b.append((cur[4] - cur[7], cur[11]))
        gaps.append((cur[0].min() - t0, cur[10].max() - t0))
print(f"{args.config}: {G} CTAs; times in us relative to the previous launch's last CTA end (median over launches)")
for nm in names:
    a = np.array(acc[nm]) / 1e3
    print(f"  {nm:6s} min {np.median(a.min(1)):7.2f}  median {np.median(np.median(a, 1)):7.2f}  max {np.median(a.max(1)):7.2f}")
g = np.array(gaps) / 1e3
print(f"  launch period (last end -> last end) median {np.median(g[:, 1]):.2f} us; first CTA start after previous end {np.median(g[:, 0]):.2f} us")
bdur = np.array([p[0] for p in per_cta_b]) / 1e3
sm = per_cta_b[0][1]
order = np.argsort(sm)
md = np.median(bdur, 0)
print("  phase-B duration per CTA (rel1 -> arr2), median over launches: min %.2f median %.2f max %.2f" % (md.min(), np.median(md), md.max()))
half = sm.max() // 2
lo, hi = md[sm <= half], md[sm > half]
print(f"  by SM id: <= {half}: mean {lo.mean():.2f}  > {half}: mean {hi.mean():.2f}")
print("  per CTA (sorted by smid) B us:", " ".join(f"{sm[i]}:{md[i]:.1f}" for i in order))
