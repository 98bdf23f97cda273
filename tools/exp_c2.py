"""Back-to-back device-resident apply time of one config under the current
environment knobs, plus the persistent kernel's phase split (stamps of
isolated applies, warm L2). Used for A/B runs of kernel variants.

    TBT_PREFETCH=1 python tools/exp_c2.py --config C2
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--tag", default="")
args = ap.parse_args()
cfg = CONFIGS[args.config]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
st = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
n = op.size()
x = torch.randn(n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(20):
    op.apply_device(x.data_ptr(), y.data_ptr())
st.synchronize()
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.n):
        op.apply_device(x.data_ptr(), y.data_ptr())
    e1.record(st)
    st.synchronize()
    res.append(e0.elapsed_time(e1) / args.n * 1e3)
op.phase_times(True)
rows = []
for _ in range(50):
    op.apply_device(x.data_ptr(), y.data_ptr())
    st.synchronize()
    rows.append(op.phase_times(True))
op.phase_times(False)
med = [statistics.median(r[i] for r in rows) for i in range(13)]
ph = " ".join(f"{v:5.2f}" for v in med[:5])
spread = " ".join(f"{med[5 + k] - med[9 + k]:4.2f}" for k in range(4))
print(f"{args.tag:24s} {args.config} b2b {min(res):6.2f} us  phases [{ph}]  barrier spreads [{spread}]", flush=True)
