python tools/bench_configs.py --configs C5 --no-cpu 2>&1 | python -c "import json,sys; [print(r['config'], r['pow2']['gmres']) for r in map(json.loads, sys.stdin)]"
for cfg in C3 C4; do for mode in default cols; do echo "== $cfg $mode"; if [ $mode = cols ]; then export TBT_GMRES=cols; else unset TBT_GMRES; fi; python tools/bench_configs.py --configs $cfg --no-cpu 2>&1 | python -c "import json,sys; [print(r['config'], r['pow2']['gmres']) for r in map(json.loads, sys.stdin)]"; done; done
unset TBT_GMRES
python -m pytest tests -m gpu -q -k "gmres" 2>&1 | tail -2
