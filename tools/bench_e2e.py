"""e2e apply through the C ABI with host buffers: pinned (zero-copy path)
vs pageable (staged copies)."""
import ctypes as C
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402
from paper_2506_04710_b200._lib import TBT_HOST, lib  # noqa: E402
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg))
x = np.asarray(gen.rhs_normal(cfg.n, 1, 3)[:, 0]).copy()
ref = op.apply(x)
for label, xh, yh in [("pinned", torch.from_numpy(x.copy()).pin_memory(), torch.empty(cfg.n, dtype=torch.complex128).pin_memory()),
                      ("pageable", torch.from_numpy(x.copy()), torch.empty(cfg.n, dtype=torch.complex128))]:
    for _ in range(5):
        lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
    n = 300
    t0 = time.perf_counter()
    for _ in range(n):
        lib().tbt_apply(op._h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()), 1, TBT_HOST)
    dt = (time.perf_counter() - t0) / n
    err = np.linalg.norm(yh.numpy() - ref) / np.linalg.norm(ref)
    print(f"{label}: {dt*1e6:.1f} us per e2e apply ({1/dt:.0f}/s), rel diff vs staged {err:.1e}")
