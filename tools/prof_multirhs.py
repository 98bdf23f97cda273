"""Device-resident batched applies of an nx x ny, m, nrhs operator (not a BASELINE config):
    python tools/prof_multirhs.py 32 32 64 64
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import Config, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402

nx, ny, m, k = (int(a) for a in sys.argv[1:5])
cfg = Config("X", nx, ny, m, k, 8, 5, "normal", 50)
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=k)
st = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
torch.cuda.set_stream(st)
x = torch.from_numpy(np.asfortranarray(gen.rhs_normal(cfg.n, k, 3)).T.copy()).cuda()
y = torch.empty_like(x)
for _ in range(3):
    op.apply_device(x.data_ptr(), y.data_ptr(), k)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    op.apply_device(x.data_ptr(), y.data_ptr(), k)
e.record()
e.synchronize()
ms = s.elapsed_time(e) / 10
print(f"{nx}x{ny} m={m} nrhs={k}: {ms:.3f} ms per batched apply, {k / ms * 1e3:.0f} column-matvecs/s")
