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

from paper_2506_04710_b200 import CONFIGS, Config, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--nocorr", action="store_true")
ap.add_argument("--embed", default="pow2")
args = ap.parse_args()
EXTRA = {"G48": Config("G48", 48, 48, 96, 1, 8, 5, "normal", 50), "G40": Config("G40", 40, 24, 64, 1, 8, 6, "normal", 50)}
cfg = CONFIGS[args.config] if args.config in CONFIGS else EXTRA[args.config]
rep = ToeplitzRep.synthetic(cfg)
if args.nocorr:
    rep.correction = None
op = ToeplitzMatvec(rep, max_nrhs=cfg.nrhs, embed=args.embed)
_st = torch.cuda.Stream()
op.set_stream(_st.cuda_stream)
torch.cuda.set_stream(_st)
K = cfg.nrhs
x = torch.from_numpy(np.asfortranarray(gen.rhs_normal(cfg.n, K, 3)).T.copy()).cuda()  # column-major n x K
y = torch.empty_like(x)
for _ in range(args.iters):
    op.apply_device(x.data_ptr(), y.data_ptr(), K)
torch.cuda.synchronize()
print("ok", args.config, float(y.abs().sum()))

if K > 1:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        op.apply_device(x.data_ptr(), y.data_ptr(), K)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 10
    flops = 8.0 * cfg.m * cfg.m * K * op.info().bins
    print(f"nrhs={K}: {ms:.3f} ms per batched apply, {K / ms * 1e3:.0f} column-matvecs/s, "
          f"bin-product {flops / (ms * 1e-3) / 1e12:.1f} TFLOP/s equivalent over the whole apply")
    sys.exit(0)
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
