"""Per-kernel timeline of tbt_apply_many (TBT_CTATRACE=1, TBT_MANY=direct):
the last 8 applies of a 16-vector pinned batch, each relative to the
previous apply's last CTA end: first CTA start, programmatic-wait end,
phase B (barrier 1 release -> barrier 2 last arrival), C2 end."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("TBT_CTATRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402

cfg = CONFIGS["C2"]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
nb = 16
xs = torch.from_numpy(np.ascontiguousarray(gen.rhs_normal(cfg.n, nb, 77).T)).pin_memory()
ys = torch.empty_like(xs).pin_memory()
for _ in range(3):
    op.apply_many_ptr(xs.data_ptr(), ys.data_ptr(), nb)
cnt, tr = op.cta_trace()
G = torch.cuda.get_device_properties(0).multi_processor_count
tr = tr[:, :, :G].astype(np.int64)
order = sorted(range(8), key=lambda k: tr[k][0].min())
print("apply  start    pdl  rel1(B start) arr2max(B end)  C2end   (us rel. to previous apply's last end)")
for i in range(1, 8):
    p, c = tr[order[i - 1]], tr[order[i]]
    t0 = p[10].max()
    print(f"{i:4d} {(c[0].min() - t0) / 1e3:7.2f} {(c[1].max() - t0) / 1e3:6.2f} {(c[7].max() - t0) / 1e3:8.2f} "
          f"{(c[4].max() - t0) / 1e3:10.2f} {(c[10].max() - t0) / 1e3:9.2f}")
