# Warp-synchronous line groups in the cluster 2-D transforms: parity with
# small batch chunks forced, and C3 timing per (CL, BC).
mkdir -p gpurun_out
TBT_FFT2D=4,4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3 or smooth or multi_rhs" 2>&1 | tail -2
for f in "" "4,4" "4,2" "2,4" "1,4"; do
  echo "== smooth fft2d=$f"
  TBT_FFT2D=$f timeout 300 python tools/prof_apply.py --config C3 --embed smooth 2>&1 | tail -1
done
for f in "" "8,4" "4,4"; do
  echo "== pow2 fft2d=$f"
  TBT_FFT2D=$f timeout 300 python tools/prof_apply.py --config C3 2>&1 | tail -1
done
