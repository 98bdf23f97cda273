timeout 900 python -m pytest tests -m gpu -q -x -k "concurrent or apply_many or env_paths or smoke or gmres" 2>&1 | tail -3
python tools/exp_c2.py --tag single-ctx
python tools/exp_gmres.py --tag lagged
