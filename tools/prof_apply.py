"""Small driver for ncu / sanitizer runs: N device-resident applies of a
config (no oracle, no torch kernels in between).

    python tools/prof_apply.py --config C2 --iters 5
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--nocorr", action="store_true")
args = ap.parse_args()
cfg = CONFIGS[args.config]
rep = ToeplitzRep.synthetic(cfg)
if args.nocorr:
    rep.correction = None
op = ToeplitzMatvec(rep)
_st = torch.cuda.Stream()
op.set_stream(_st.cuda_stream)
torch.cuda.set_stream(_st)
x = torch.from_numpy(np.asarray(gen.rhs_normal(cfg.n, 1, 3)[:, 0]).copy()).cuda()
y = torch.empty_like(x)
for _ in range(args.iters):
    op.apply_device(x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
print("ok", args.config, float(y.abs().sum()))

if "--phases" in sys.argv or True:
    import statistics
    op.phase_times(True)
    ph = []
    for _ in range(20):
        op.apply_device(x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        ph.append(op.phase_times(True))
    op.phase_times(False)
    print("phases_us", [round(statistics.median(p[i] for p in ph), 2) for i in range(5)])
    print("barrier latest arrival", [round(statistics.median(p[i] for p in ph), 2) for i in range(5, 9)])
    print("barrier earliest arrival", [round(statistics.median(p[i] for p in ph), 2) for i in range(9, 13)])
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(100):
        op.apply_device(x.data_ptr(), y.data_ptr())
    e.record(); e.synchronize()
    print("us_per_apply_back_to_back", s.elapsed_time(e) * 10)
