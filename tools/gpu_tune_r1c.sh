# Round-1 tuning sweep (device-resident timing): persistent DMMA GEMM (C3),
# L2 prefetch of the spectrum during the forward transforms (TBT_DEV_L2="MB,at").
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "multi_rhs or c3 or many_columns" 2>&1 | tail -2
timeout 300 python tools/prof_apply.py --config C3 --embed smooth 2>&1 | tail -1
timeout 300 python tools/prof_apply.py --config C3 2>&1 | tail -1
for v in "0,0" "24,1" "48,1" "80,1" "32,0"; do
  echo "== TBT_DEV_L2=$v"
  TBT_DEV_L2=$v timeout 120 python tools/prof_phases.py --config C2 --n 50 2>&1 | tail -6
  TBT_DEV_L2=$v timeout 200 python bench.py --steps 2000 --warmup 20 --no-cpu --no-gmres 2>gpurun_out/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step']*1e3, d['roofline']['frac'], d['roofline']['phase_us'])" || tail -3 gpurun_out/err.txt
done
