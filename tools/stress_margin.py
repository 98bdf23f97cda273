"""Repeat margin applies / diagonals against the oracle (flake hunt)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from paper_2506_04710_b200 import ToeplitzMatvec, gen  # noqa: E402
from test_margin import rep_with_margin  # noqa: E402

if "--torch" in sys.argv:
    import torch
    print("torch cuda", torch.cuda.is_available())
bad = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20):
    for k in (1, 3):
        rep = rep_with_margin(8, 6, 64, [3, 5, 2, 4, 64, 6, 1, 7, 2])
        op = ToeplitzMatvec(rep, max_nrhs=k)
        o = oracle.Oracle.from_rep(rep)
        X = gen.rhs_normal(o.n, k, 11 + trial)
        Y = op.apply(X if k > 1 else X[:, 0]).reshape(o.n, k)
        for c in range(k):
            ref = o.apply(np.ascontiguousarray(X[:, c]))
            errA = np.linalg.norm(Y[:o.nA, c] - ref[:o.nA]) / np.linalg.norm(ref[:o.nA])
            errM = np.linalg.norm(Y[o.nA:, c] - ref[o.nA:]) / np.linalg.norm(ref[o.nA:])
            if not max(errA, errM) <= 1e-11:
                bad += 1
                print("BAD apply", trial, k, c, errA, errM, "nanA", int(np.isnan(Y[:o.nA, c]).sum()),
                      "nanM", int(np.isnan(Y[o.nA:, c]).sum()), flush=True)
        ya = op.applyA(np.ascontiguousarray(X[:o.nA, 0]))
        ea = np.linalg.norm(ya - o.applyA(np.ascontiguousarray(X[:o.nA, 0]))) / np.linalg.norm(ya)
        if not ea <= 1e-11:
            bad += 1
            print("BAD applyA", trial, k, ea, flush=True)
        d = op.diagonal()
        if not np.allclose(d, o.diagonal(), rtol=1e-14, atol=0):
            bad += 1
            print("BAD diag", trial, k, np.max(np.abs(d - o.diagonal())), flush=True)
        del op
# same shape without margin: A part alone
from paper_2506_04710_b200 import Config, ToeplitzRep  # noqa: E402
for corr in (False, True):
    rep = ToeplitzRep.synthetic(Config("x", 8, 6, 64, 1, 2 if corr else -1, 3, "normal", 20, scale=0.1 if corr else 0.0))
    op = ToeplitzMatvec(rep)
    o = oracle.Oracle.from_rep(rep)
    x = gen.rhs_normal(o.n, 1, 5)[:, 0]
    y = op.apply(x)
    print("no-margin corr", corr, "nan", int(np.isnan(y).sum()), np.linalg.norm(y - o.apply(x)) / np.linalg.norm(o.apply(x)))
print("bad", bad)
