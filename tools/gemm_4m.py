"""3M vs 4M complex DMMA GEMM for the many-RHS bin product (C3). Run once per
form (TBT_GEMM is read once per process):

    python tools/gemm_4m.py            # 3M (default)
    TBT_GEMM=4m python tools/gemm_4m.py

Prints per embedding: apply ms, bin-product ms (tbt_set_timing), and the
relative error of 8 sampled columns against the oracle (max and mean)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen  # noqa: E402

cfg = CONFIGS["C3"]
rep = ToeplitzRep.synthetic(cfg)
o = oracle.Oracle.from_rep(rep)
K = cfg.nrhs
Xh = gen.rhs_normal(cfg.n, K, 3)
cols = list(range(0, K, K // 8))[:8]
refs = [o.apply(np.ascontiguousarray(Xh[:, c])) for c in cols]
for embed in ("smooth", "pow2"):
    op = ToeplitzMatvec(rep, max_nrhs=K, embed=embed)
    stream = torch.cuda.Stream()
    op.set_stream(stream.cuda_stream)
    x = torch.from_numpy(np.ascontiguousarray(Xh.T)).cuda()
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply_device(x.data_ptr(), y.data_ptr(), K)
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record(stream)
    for _ in range(n):
        op.apply_device(x.data_ptr(), y.data_ptr(), K)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    op.set_timing(True)
    for _ in range(n):
        op.apply_device(x.data_ptr(), y.data_ptr(), K)
    bp, cnt = op.timing_read()
    op.set_timing(False)
    Y = y.cpu().numpy().T
    errs = [float(np.linalg.norm(Y[:, c] - r) / np.linalg.norm(r)) for c, r in zip(cols, refs)]
    print(json.dumps({"form": os.environ.get("TBT_GEMM", "3m"), "embed": embed, "apply_ms": ms,
                      "binprod_ms": bp / max(cnt, 1), "rel_err_max": max(errs), "rel_err_mean": float(np.mean(errs))}),
          flush=True)
    op.close()
