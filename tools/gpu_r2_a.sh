mkdir -p gpurun_out
free -g | head -2
timeout 900 python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
/usr/bin/time -f "bench wall %e s" timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -1 gpurun_out/r2a_bench.err
python -c "import json; d=json.loads(open('gpurun_out/r2a_bench.json').read()); print(d['value'], d['roofline']['frac'], d['roofline'].get('k3_phase_frac'), d['e2e']['value'], d['cpu_baseline']); print(json.dumps(d['large_configs'])[:3000])"
/usr/bin/time -f "ref wall %e s" timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err; tail -1 gpurun_out/r2a_ref.err; head -c 600 gpurun_out/r2a_ref.json
