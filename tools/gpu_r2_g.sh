mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_margin.py tests/test_dist_loopback.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --configs G48,G40 --no-cpu 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2g_g48.csv python tools/prof_apply.py --config G48 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/r2g_g48.csv
