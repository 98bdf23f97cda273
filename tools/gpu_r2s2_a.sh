# Session-2 check of HEAD: GPU suite, smoke, bench (both arms).
mkdir -p gpurun_out/s2a
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
start=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s2a/gpu_tests.log; echo "gpu suite $(( $(date +%s) - start )) s"; tail -3 gpurun_out/s2a/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/s2a/bench.json 2> gpurun_out/s2a/bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/s2a/bench_reference.json 2> gpurun_out/s2a/bench_reference.err; echo "ref rc $?"
