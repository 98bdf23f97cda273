# LS step: L rows prefetched under pass 1. GMRES parity + C2 LS timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_margin.py -m gpu -q -x -k "gmres or schur" 2>&1 | tail -2
for i in 1 2; do TBT_LSPROF=1 timeout 200 python tools/bench_gmres.py C2 200 2>&1 | grep -v "^$" | tail -2; done
