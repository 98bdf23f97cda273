# DMMA GEMM: padded transposed A chunk (TBT_GEMM_TPAD) A/B on C3, + parity.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_margin.py -m gpu -q -x -k "multi_rhs or c3 or many_columns or schur" 2>&1 | tail -2
for i in 1 2; do
for t in 0 1; do
  echo "== TPAD=$t"
  TBT_GEMM_TPAD=$t timeout 300 python tools/prof_apply.py --config C3 --embed smooth 2>&1 | tail -1
  TBT_GEMM_TPAD=$t timeout 300 python tools/prof_apply.py --config C3 2>&1 | tail -1
done
done
./tools/fp64test 2>&1 | tail -8
