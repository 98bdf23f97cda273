"""Small run over every kernel path, for compute-sanitizer (one tool per
call): persistent apply, fused and line-pass transforms, DMMA GEMM, smooth
embedding, correction, GMRES (both orthogonalisations, multi-column), and the
one-rank NCCL path."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2506_04710_b200 import (CONFIGS, Config, SolverOptions, ToeplitzMatvec, ToeplitzRep,  # noqa: E402
                                   dist_unique_id, gen)


def rep(nx, ny, m, seed=1):
    return ToeplitzRep.synthetic(Config("s", nx, ny, m, 1, 4, seed, "normal", 20))


def run():
    r = ToeplitzRep.synthetic(CONFIGS["C2"])
    op = ToeplitzMatvec(r)
    x = gen.rhs_normal(op.sizeA(), 1, 1)[:, 0]
    op.apply(x)
    op.gmres(x, SolverOptions(tol=1e-8, maxIter=12, restart=5), raise_on_fail=False)
    op.gmres(x, SolverOptions(tol=1e-8, maxIter=12, restart=5, orthog=0), raise_on_fail=False)
    for shape, k, embed in [((4, 4, 24), 1, "pow2"), ((6, 5, 64), 9, "pow2"), ((18, 9, 8), 3, "smooth"),
                            ((5, 3, 128), 10, "pow2")]:
        o2 = ToeplitzMatvec(rep(*shape), max_nrhs=k, embed=embed)
        X = gen.rhs_normal(o2.sizeA(), k, 2)
        o2.apply(X if k > 1 else X[:, 0])
        o2.applyA(X if k > 1 else X[:, 0])
        o2.gmres(X, SolverOptions(tol=1e-9, maxIter=20, restart=6), raise_on_fail=False)
    os.environ["TBT_FFT"] = "passes"
    o3 = ToeplitzMatvec(rep(7, 9, 64), max_nrhs=2)
    o3.apply(gen.rhs_normal(o3.sizeA(), 2, 3))
    del os.environ["TBT_FFT"]
    o4 = ToeplitzMatvec(rep(6, 5, 64), dist=(1, 0, dist_unique_id()))
    o4.apply(gen.rhs_normal(o4.sizeA(), 1, 4)[:, 0])
    print("sanitize suite ok")


if __name__ == "__main__":
    run()
