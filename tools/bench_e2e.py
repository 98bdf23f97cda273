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

# Pure transfer cost of one step's vectors (pinned, CUDA events).
xd = torch.empty(cfg.n, dtype=torch.complex128, device="cuda")
xp = torch.from_numpy(x.copy()).pin_memory()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        xd.copy_(xp, non_blocking=True)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(s)
    for _ in range(100):
        xd.copy_(xp, non_blocking=True)
    e1.record(s)
    for _ in range(100):
        xp.copy_(xd, non_blocking=True)
    e2.record(s)
    e2.synchronize()
print(f"pinned H2D {cfg.n * 16 / 1e6:.2f} MB: {e0.elapsed_time(e1) * 10:.1f} us, D2H: {e1.elapsed_time(e2) * 10:.1f} us")
