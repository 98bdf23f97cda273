"""Phase split of the persistent apply (CTA 0 %globaltimer stamps) and the
grid-barrier arrival spread: for barrier k, the earliest and latest CTA
arrival relative to CTA 0's phase start, and CTA 0's release.

    python tools/prof_phases.py [--config C2] [--n 50]
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--n", type=int, default=50)
args = ap.parse_args()
cfg = CONFIGS[args.config]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
st = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
n = op.size()
x = torch.randn(n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(5):
    op.apply_device(x.data_ptr(), y.data_ptr())
st.synchronize()
op.phase_times(True)
rows = []
for _ in range(args.n):
    op.apply_device(x.data_ptr(), y.data_ptr())
    st.synchronize()
    rows.append(op.phase_times(True))
op.phase_times(False)
med = [statistics.median(r[i] for r in rows) for i in range(13)]
names = ["A1 rows", "A2 cols", "B binprod", "C1 inv cols", "C2 inv rows"]
for k in range(5):
    line = f"{names[k]:12s} {med[k]:7.2f} us"
    if k < 4:
        line += f"   barrier {k}: first arrival {med[9 + k]:6.2f}  last arrival {med[5 + k]:6.2f}  release {med[k]:6.2f}"
    print(line)
print(f"total {sum(med[:5]):.2f} us")
