# New GPU property tests, dist tests, and the bench line with the sharded C4 block.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_dist.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu > gpurun_out/b_sharded.json 2> gpurun_out/b_sharded.err; python -c "import json; d=json.load(open('gpurun_out/b_sharded.json')); print(d['value'], d['sharded'])" || tail -5 gpurun_out/b_sharded.err
