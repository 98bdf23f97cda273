# L2 persisting access-policy window over the Krylov basis (TBT_L2_PERSIST).
mkdir -p gpurun_out
for k in 0 1 0 1; do
  echo "== TBT_L2_PERSIST=$k"
  TBT_L2_PERSIST=$k TBT_LSPROF=1 timeout 200 python tools/bench_gmres.py C2 200 2>&1 | grep -v "^$" | grep -v "^C2" | tail -4
done
TBT_L2_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gmres" 2>&1 | tail -2
