# Round-1 (third session) measurement pass: tests, bench, all configs, and
# the ncu evidence of the bench's kernel — each ncu command only after the
# same command ran clean without ncu.
set -x
mkdir -p gpurun_out/ncu
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err; tail -c 600 gpurun_out/r1c_bench.json
timeout 900 python tools/bench_configs.py --out gpurun_out/r1c_configs.json > gpurun_out/r1c_configs.log 2>&1; tail -c 800 gpurun_out/r1c_configs.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-gmres > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/ncu/r1c_bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-gmres > /dev/null 2>&1
timeout 300 python tools/prof_apply.py --config C2 --iters 8 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/ncu/r1c_c2_persistent -f python tools/prof_apply.py --config C2 --iters 8 > /dev/null 2>&1
ls -la gpurun_out/ncu
