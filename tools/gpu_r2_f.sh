mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gmres_large.py tests/test_gpu_parity.py tests/test_env_paths.py -m gpu -q -x 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_gm_C5.csv python tools/prof_gmres.py C5 50 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2f_gm_C5.csv | grep -v "gatherShift\|fftPassKernel\|scatterPairs\|layoutKernel"
timeout 600 python bench.py --no-cpu --no-sharded > gpurun_out/r2f_bench.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r2f_bench.json').read()); print(d['value'], d['gmres']['ms_per_iteration']); [print(k, v['ms_per_apply'], v['gmres']) for k,v in d['large_configs'].items()]"
