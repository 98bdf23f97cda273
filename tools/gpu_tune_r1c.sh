# Default bench run (with the sharded C4 block incl. distributed GMRES).
mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python bench.py > gpurun_out/b_full.json 2> gpurun_out/b_full.err
echo "bench wall s: $(( $(date +%s) - start ))"
python -c "import json; d=json.loads(open('gpurun_out/b_full.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['gmres']['ms_per_iteration']); print(d['sharded'])" || tail -5 gpurun_out/b_full.err
