# Late-round-1 recaptures (one GPU; every command ran clean without ncu first):
# the persistent apply after the slab padding / PDL changes, and the fused
# single-column margin kernels.
set -x
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/ncu/r1b_c2_persistent -f python tools/prof_apply.py --config C2 --iters 8 > /dev/null 2>&1
$NCU -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/ncu/r1b_c4_persistent -f python tools/prof_apply.py --config C4 --iters 8 > /dev/null 2>&1
$NCU -k regex:"sideFused|rowFused|cornerFused" -s 6 -c 3 -o gpurun_out/ncu/r1b_c4_margin -f python tools/bench_margin.py --config C4 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/ncu/r1b_bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-gmres > /dev/null 2>&1
ls -la gpurun_out/ncu
