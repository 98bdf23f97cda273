mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_env_paths.py tests/test_gmres_large.py tests/test_ref_pin.py tests/test_ztoe1.py -m gpu -q --durations=8 2>&1 | tail -25
