# Session-3 check: full GPU suite, smoke, both bench arms on the current tree.
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
start=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6; echo "gpu suite $(( $(date +%s) - start )) s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/s3/bench.json').read()); print(d['value'], d['ms_per_step'], d['roofline'], d['e2e'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/s3/bench_reference.json 2> gpurun_out/s3/bench_reference.err; echo "ref rc $?"; head -c 600 gpurun_out/s3/bench_reference.json
