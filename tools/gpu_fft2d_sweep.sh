for v in 4,16 2,16 3,16 6,16 4,8 6,8 3,8 2,8 6,4 4,4; do
  echo "== $v"; TBT_FFT2D=$v python tools/prof_apply.py --config C3 --embed smooth --iters 3 2>&1 | grep "ms per"
  TBT_FFT2D=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fft2d -c 4 --csv python tools/prof_apply.py --config C3 --embed smooth --iters 2 2>/dev/null | grep -o '"fft2dKernel<[^"]*".*' | awk -F'","' '{print $1, $NF}' | tail -2
done
