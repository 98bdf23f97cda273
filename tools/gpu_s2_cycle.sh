# Restart-cycle kernel + plain PDL launches: parity subset, GMRES timing, apply b2b.
timeout 900 python -m pytest tests -m gpu -q -x -k "gmres or env_paths or smoke or persistent" 2>&1 | tail -5
python tools/exp_c2.py --tag plain+pdl
TBT_COOP=1 python tools/exp_c2.py --tag coop=1
timeout 600 python bench.py --steps 2000 --no-cpu --no-sharded > gpurun_out/s2_cycle_bench.json 2>gpurun_out/s2_cycle_bench.err; echo "bench rc $?"
python -c "
import json;d=json.load(open('gpurun_out/s2_cycle_bench.json'));print('value',d['value'],'gmres',d['gmres']['ms_per_iteration'])
for k,v in d.get('large_configs',{}).items(): print(k, v['ms_per_apply'], v['gmres']['ms_per_iteration'])"
TBT_LSPROF=1 timeout 300 python tools/prof_gmres.py C2 200
