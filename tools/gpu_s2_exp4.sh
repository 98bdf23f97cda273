timeout 900 python -m pytest tests -m gpu -q -x -k "gmres or env_paths or smoke or persistent or ref_pin" 2>&1 | tail -3
python tools/exp_c2.py --tag apply
for r in 1 2; do
python tools/exp_gmres.py --tag lagged
TBT_GMRES=nolag python tools/exp_gmres.py --tag nolag
done
TBT_LSPROF=1 python tools/exp_gmres.py --tag lagged 2>&1 | tail -2
