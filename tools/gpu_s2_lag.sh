timeout 900 python -m pytest tests -m gpu -q -x -k "gmres or env_paths or smoke or persistent or ref_pin" 2>&1 | tail -5
for r in 1 2; do
python tools/exp_gmres.py --tag cycle-lagged
TBT_GMRES=graph python tools/exp_gmres.py --tag graph
done
TBT_LSPROF=1 python tools/exp_gmres.py --tag cycle-lagged 2>&1 | tail -2
