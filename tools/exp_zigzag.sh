# Zig-zag pair order experiment: back-to-back apply and GMRES per-iteration
# time. TBT_ZIGZAG = 0 off, 1 alternate (evict_first); TBT_ZZTAIL = % of a
# CTA's items (time order, last) loaded evict_last.
mkdir -p gpurun_out/zz
run() {
  env $1 timeout 600 python tools/bench_configs.py --configs C2,G40 --no-cpu --out gpurun_out/zz/r.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/zz/r.json'))
print('$1', ' '.join(f\"{c['config']}: apply {c['pow2']['ms_per_apply']*1e3:.1f}us gmres {c['pow2']['gmres']['ms_per_iteration']*1e3:.1f}us\" for c in d))"
}
run TBT_ZIGZAG=0
run TBT_ZIGZAG=1
for t in 15 30 45 60; do run "TBT_ZIGZAG=1 TBT_ZZTAIL=$t"; done
run TBT_ZIGZAG=0
