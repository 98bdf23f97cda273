timeout 1200 python -m pytest tests/test_env_paths.py tests/test_semisparse.py tests/test_ztoe1.py tests/test_margin.py tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -15
