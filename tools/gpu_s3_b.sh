mkdir -p gpurun_out/s3
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_env_paths.py tests/test_gmres_large.py tests/test_ref_pin.py tests/test_concurrent_contexts.py -m gpu -q -x 2>&1 | tail -3
for z in 1 0; do
  TBT_ZIGZAG=$z timeout 600 python tools/bench_configs.py --configs C1,C2,G40,C4 --no-cpu --out gpurun_out/s3/zz$z.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/s3/zz$z.json'))
print('ZZ=$z', ' '.join(f\"{c['config']}: apply {c['pow2']['ms_per_apply']*1e3:.1f}us gmres {c['pow2']['gmres']['ms_per_iteration']*1e3:.1f}us\" for c in d))"
done
