# C3 GEMM as two 4-warp CTAs per SM: parity, apply time, kernel time.
timeout 900 python -m pytest tests/test_env_paths.py -m gpu -q -k "GEMM" 2>&1 | tail -3
for g in wide pair2 pair3; do echo "GEMM $g"; TBT_GEMM=$g python tools/prof_apply.py --config C3 --embed smooth --iters 4 | tail -1; TBT_GEMM=$g python tools/prof_apply.py --config C3 --embed pow2 --iters 4 | tail -1; done
for g in wide pair2 pair3; do
TBT_GEMM=$g ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"binprodGemm" -s 4 -c 1 --csv python tools/prof_apply.py --config C3 --embed smooth --iters 4 2>/dev/null | grep -E "binprod" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-60,100-200
done
