# Round-2 baseline: GPU suite, smoke, bench both arms.
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
cat gpurun_out/r2_bench.json | head -c 3000
timeout 300 python tools/bench_configs.py > gpurun_out/r2_configs.json 2> gpurun_out/r2_configs.err
tail -c 2000 gpurun_out/r2_configs.json
