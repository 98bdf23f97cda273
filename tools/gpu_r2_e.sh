mkdir -p gpurun_out
for cfg in C4 C5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_gm_${cfg}.csv python tools/prof_gmres.py $cfg 50 > /dev/null 2>&1
  echo "== $cfg"; python tools/launch_summary.py gpurun_out/r2e_gm_${cfg}.csv
done
