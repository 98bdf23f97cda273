timeout 900 python -m pytest tests -m gpu -q -x -k "apply_many or env_paths or smoke" 2>&1 | tail -3
for r in 1 2; do
python tools/exp_e2e.py --tag flags
TBT_MANY=events python tools/exp_e2e.py --tag events
done
