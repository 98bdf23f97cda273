"""Phase split of the zero-copy e2e apply (persistent kernel reading x from /
writing y to pinned host memory) vs the device-resident apply."""
import ctypes as C
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402
from paper_2506_04710_b200._lib import TBT_HOST, lib  # noqa: E402

cfg = CONFIGS["C2"]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg))
x = np.asarray(gen.rhs_normal(cfg.n, 1, 3)[:, 0]).copy()
xh = torch.from_numpy(x.copy()).pin_memory()
yh = torch.empty(cfg.n, dtype=torch.complex128).pin_memory()
xd, yd = xh.cuda(), torch.empty(cfg.n, dtype=torch.complex128, device="cuda")
for label, a, b, where in [("zero-copy host", xh, yh, TBT_HOST), ("device", xd, yd, 1)]:
    for _ in range(10):
        lib().tbt_apply(op._h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), 1, where)
    op.phase_times(True)
    ph = []
    for _ in range(50):
        lib().tbt_apply(op._h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), 1, where)
        torch.cuda.synchronize()
        ph.append(op.phase_times(True))
    op.phase_times(False)
    print(label, "phases_us", [round(statistics.median(p[i] for p in ph), 2) for i in range(5)])
