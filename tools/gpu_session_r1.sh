set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; tail -c 1500 gpurun_out/configs.log
