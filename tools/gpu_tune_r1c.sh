# Dynamically scheduled persistent DMMA GEMM: parity + C3 timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_margin.py -m gpu -q -x -k "multi_rhs or c3 or smooth or many_columns or schur" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python tools/prof_apply.py --config C3 --embed smooth 2>&1 | tail -1
timeout 300 python tools/prof_apply.py --config C3 2>&1 | tail -1
done
timeout 300 python tools/bench_gmres.py C3 50 smooth 2>&1 | tail -2
