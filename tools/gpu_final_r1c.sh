# End-of-session check: GPU suite, smoke, both bench arms (stdout must be
# exactly one JSON line each).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench stdout lines: $(wc -l < gpurun_out/final_bench.json)"
python -c "import json; d=json.loads(open('gpurun_out/final_bench.json').read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['gmres']['ms_per_iteration'], d['sharded']['ms_per_matvec'], d['clocks'])"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
echo "ref stdout lines: $(wc -l < gpurun_out/final_ref.json)"; head -c 300 gpurun_out/final_ref.json
