# Per-device launch-attribute setup: the whole GPU suite.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
