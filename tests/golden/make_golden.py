"""Generates tests/golden/ref_fft.npz from the REFERENCE's own fftInPlace
(/root/reference/proj/src/fft.cpp compiled by oracle/Makefile into
oracle/_ref/libref_fft.so). Run in the dev container, where the reference
tree exists; the .npz is committed so the GPU box (no /root/reference)
checks against it too.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
import oracle  # noqa: E402

rng = np.random.default_rng(20250604)
out = {}
for n in [1, 2, 4, 8, 16, 32, 64, 128, 256]:
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    out[f"in_{n}"] = x
    out[f"fwd_{n}"] = oracle.ref_fft(x, False)
    out[f"inv_{n}"] = oracle.ref_fft(x, True)
out["next_pow2"] = np.array([[k, oracle.ref_lib().ref_next_pow2(k)] for k in range(1, 300)], dtype=np.int64)
np.savez_compressed(REPO / "tests" / "golden" / "ref_fft.npz", **out)
print("wrote", REPO / "tests" / "golden" / "ref_fft.npz")
