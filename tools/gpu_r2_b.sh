mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_loopback.py tests/test_dist.py -m gpu -q -x 2>&1 | tail -15
start=$(date +%s); timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench wall $(( $(date +%s) - start )) s"
tail -3 gpurun_out/r2b_bench.err
python -c "import json; d=json.loads(open('gpurun_out/r2b_bench.json').read()); print(d['value'], d['roofline']['frac'], d['roofline'].get('k3_phase_frac'), d['e2e']['value'], d['cpu_baseline']); print(json.dumps(d['large_configs'])[:3000]); print(d['sharded'])"
start=$(date +%s); timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err; echo "ref wall $(( $(date +%s) - start )) s"; head -c 800 gpurun_out/r2b_ref.json
