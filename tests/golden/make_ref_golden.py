"""Writes tests/golden/ref_pin.npz: outputs of the reference ITSELF
(oracle/_ref/libref_linsolve.so, the reference's linsolve.cpp / toeplitz.cpp
/ fft.cpp compiled unchanged against oracle/eigen_shim) on seeded inputs,
so tests/test_ref_pin.py::test_golden_reference_outputs pins the oracle
where that library is absent.

    python tests/golden/make_ref_golden.py
"""
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

import oracle  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, gen  # noqa: E402
from test_ref_pin import random_blocks  # noqa: E402
from ztoe1_writer import write_ztoe1  # noqa: E402


def main():
    oracle.bind_inputs()
    out = {}
    with tempfile.TemporaryDirectory() as td:
        cfg = CONFIGS["C1"]
        e = [0] * 9
        e[4] = cfg.m
        p = Path(td) / "c1.ztoe1"
        write_ztoe1(str(p), cfg.nx, cfg.ny, e, gen.blocks_raw(cfg.nx, cfg.ny, cfg.m, cfg.seed))
        R = oracle.RefOperator(p)
        x = gen.rhs_normal(cfg.n, 1, 7)[:, 0]
        out["c1_x"], out["c1_y"] = x, R.applyA(x)
        out["c1_diag"] = R.diagonal()
        b = gen.rhs_normal(cfg.n, 1, cfg.seed)[:, 0]
        r = R.gmres(b, tol=cfg.tol, max_iter=2000, restart=cfg.restart)
        out["c1_b"], out["c1_gmres_x"] = b, r["x"]
        out["c1_gmres_iterations"] = np.int64(r["iterations"])
        out["c1_gmres_residual"] = np.float64(r["residual"])
        e = [0] * 9
        e[4] = 4
        p = Path(td) / "r.ztoe1"
        write_ztoe1(str(p), 5, 3, e, random_blocks(5, 3, 4, 534))
        R = oracle.RefOperator(p)
        xr = gen.rhs_normal(60, 1, 8)[:, 0]
        out["r_x"], out["r_y"] = xr, R.applyA(xr)
    np.savez_compressed(HERE / "ref_pin.npz", **out)
    print("wrote", HERE / "ref_pin.npz", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
