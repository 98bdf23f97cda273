"""e2e rates through the C ABI under the current environment knobs: one
tbt_apply(TBT_HOST) per vector (zero-copy persistent kernel + sync) and
tbt_apply_many over 64 pinned host vectors (copies overlapped).

    TBT_COOP=1 python tools/exp_e2e.py --tag coop
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402
from paper_2506_04710_b200._lib import TBT_HOST, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--tag", default="")
args = ap.parse_args()
cfg = CONFIGS[args.config]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
st = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
xh = torch.from_numpy(np.asarray(gen.rhs_normal(cfg.n, 1, 3)[:, 0]).copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()
for _ in range(20):
    lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
single = n / (time.perf_counter() - t0)
nb = 64
xs = torch.from_numpy(np.ascontiguousarray(gen.rhs_normal(cfg.n, nb, 77).T)).pin_memory()
ys = torch.empty_like(xs).pin_memory()
op.apply_many_ptr(xs.data_ptr(), ys.data_ptr(), nb)
calls = 30
t0 = time.perf_counter()
for _ in range(calls):
    op.apply_many_ptr(xs.data_ptr(), ys.data_ptr(), nb)
many = calls * nb / (time.perf_counter() - t0)
print(f"{args.tag:12s} {args.config} e2e single {single:8.0f}/s ({1e6 / single:6.1f} us)  many {many:8.0f}/s ({1e6 / many:6.1f} us)",
      flush=True)
