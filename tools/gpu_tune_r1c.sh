# Software-pipelined column-phase FFT items: parity + phase timing (C2, C4, C5).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config_apply or c4_sampled or c5_full or apply_matches or gmres_c2" 2>&1 | tail -2
for c in C2 C4; do
  echo "== $c"
  timeout 300 python tools/prof_phases.py --config $c --n 30 2>&1 | tail -6
done
echo "== C5"
timeout 600 python tools/prof_phases.py --config C5 --n 10 2>&1 | tail -6
