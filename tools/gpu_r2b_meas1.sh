# Round-2 (second session) measurement, part 1: GPU suite, smoke, both bench
# arms, every config, the bench launch list and --set full captures of the
# C2 / C4 persistent applies and the C3 DMMA GEMM (every ncu pass after the
# same command ran clean). Part 2: tools/gpu_r2b_meas2.sh (the gpurun_out
# limit is 64 MiB per call).
mkdir -p gpurun_out/r2b
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader
start=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "gpu suite $(( $(date +%s) - start )) s"
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2b/bench_reference.json 2> gpurun_out/r2b/bench_reference.err; echo "ref rc $?"
timeout 1500 python tools/bench_configs.py --configs C1,C2,C3,C4,C5,G48,G40 --out gpurun_out/r2b/configs.json > gpurun_out/r2b/configs.log 2>&1; echo "configs rc $?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2b/bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-gmres --no-sharded --no-large > /dev/null 2>&1; echo "launches rc $?"
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/r2b/c2_persistent python tools/prof_apply.py --config C2 --iters 8 > /dev/null 2>&1; echo "c2 rc $?"
$NCU -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/r2b/c4_persistent python tools/prof_apply.py --config C4 --iters 8 > /dev/null 2>&1; echo "c4 rc $?"
$NCU -k regex:binprodGemm -s 2 -c 1 -o gpurun_out/r2b/c3_gemm python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1; echo "gemm rc $?"
du -sh gpurun_out
