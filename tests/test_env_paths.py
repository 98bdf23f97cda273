"""Every non-default product path behind an environment knob is held to the
same oracle parity as the default (tests/env_paths_check.py in a fresh
process per setting; the knobs are read once per process):

  TBT_APPLY=multi     multi-launch apply instead of the persistent kernel
  TBT_GMRES=cols      column-blocked Arnoldi for a single column
  TBT_GMRES=unfused   separate apply / Arnoldi launches (no fused epilogue)
  TBT_GMRES=nolag     fused apply + Arnoldi nodes without the lagged
                      normalisation (normalise + Givens inside each node)
  TBT_ZIGZAG=0        GMRES applies keep one bin-pair order (no alternation)
  TBT_COOP=1          every persistent apply launched cooperatively
  TBT_BINPROD=1       K3 v1 (no TMA ring), with TBT_APPLY=multi
  TBT_PDL=0           device-resident applies replayed from a CUDA graph
  TBT_FFT=passes      line-pass transforms instead of the cluster 2-D kernels
  TBT_FFT=fused       cluster 2-D kernels also for wide batches (default there:
                      register line passes)
  TBT_FFT2D=2,4       cluster 2-D transform with a forced cluster / batch split
  TBT_E2E=staged      host applies through explicit copies, not zero-copy
  TBT_MARGIN_UNFUSED=1  separate margin B / B^T kernels for one column
  TBT_GEMM=4m         4M complex DMMA GEMM for many right-hand sides
  TBT_GEMM=wide|pair2|pair3|late3  3M GEMM at m = 128 as one 8-warp CTA per
                      SM / as two 4-warp CTAs per SM with the chunk loads
                      issued ahead of the chunk (2- / 3-stage ring) or
                      between its DMMA groups with a 3-stage ring (default:
                      two 4-warp CTAs, 2-stage ring, loads between the groups)
  TBT_CORR=vec        rank-8 many-column correction on DFMA + warp shuffles
                      (corrMulti) instead of the FP64 tensor path (corrDmma)
  TBT_CORR_RPW=1|4    columns per warp of corrMulti
  TBT_DIST_CHUNKS=k   sharded apply with k overlapped exchange chunks
                      (default 2 at P > 1, 1 at P = 1)
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

SCRIPT = Path(__file__).resolve().parent / "env_paths_check.py"

CASES = [
    ({}, ["apply", "gmres", "smooth", "margin", "wide", "many"]),  # the defaults (single after multi-column applies)
    ({"TBT_FFT": "fused"}, ["wide"]),
    ({"TBT_APPLY": "multi"}, ["apply", "gmres"]),
    ({"TBT_GMRES": "cols"}, ["gmres"]),
    ({"TBT_GMRES": "unfused"}, ["gmres"]),
    ({"TBT_GMRES": "nolag"}, ["gmres"]),
    ({"TBT_ZIGZAG": "0"}, ["gmres"]),
    ({"TBT_COOP": "1"}, ["apply", "gmres"]),
    ({"TBT_BINPROD": "1", "TBT_APPLY": "multi"}, ["apply"]),
    ({"TBT_PDL": "0"}, ["apply", "gmres"]),
    ({"TBT_FFT": "passes"}, ["smooth", "apply"]),
    ({"TBT_FFT2D": "2,4"}, ["smooth"]),
    ({"TBT_E2E": "staged"}, ["apply"]),
    ({"TBT_MARGIN_UNFUSED": "1"}, ["margin"]),
    ({"TBT_GEMM": "4m"}, ["wide", "smooth"]),
    ({"TBT_GEMM": "wide"}, ["wide"]),
    ({"TBT_GEMM": "pair2"}, ["wide"]),
    ({"TBT_GEMM": "pair3"}, ["wide"]),
    ({"TBT_GEMM": "late3"}, ["wide"]),
    ({"TBT_CORR": "vec"}, ["wide"]),
    ({"TBT_CORR": "vec", "TBT_CORR_RPW": "4"}, ["wide"]),
    ({"TBT_CORR": "vec", "TBT_CORR_RPW": "1"}, ["wide"]),
    ({}, ["dist"]),
    ({"TBT_DIST_CHUNKS": "2"}, ["dist"]),
    ({"TBT_DIST_CHUNKS": "4"}, ["dist"]),
]


@pytest.mark.gpu
@pytest.mark.parametrize("env,checks", CASES, ids=[",".join(f"{k}={v}" for k, v in e.items()) or "defaults" for e, _ in CASES])
def test_env_path_parity(gpu, env, checks):
    full = dict(os.environ, **env)
    r = subprocess.run([sys.executable, str(SCRIPT), *checks], env=full, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-3000:]
    for c in checks:
        assert f"OK {c}" in r.stdout
