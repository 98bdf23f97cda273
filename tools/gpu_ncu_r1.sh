# ncu --set full captures of the top kernels (one GPU, after the same commands ran clean).
set -x
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/ncu/c2_persistent -f python tools/prof_apply.py --config C2 --iters 8 > /dev/null 2>&1
$NCU -k regex:binprodGemm -s 2 -c 1 -o gpurun_out/ncu/c3_gemm -f python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1
$NCU -k regex:corrMulti -s 2 -c 1 -o gpurun_out/ncu/c3_corr -f python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1
$NCU -k regex:fft2dKernel -s 4 -c 2 -o gpurun_out/ncu/c3_fft2d -f python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1
$NCU -k regex:lsColsDots -s 10 -c 1 -o gpurun_out/ncu/c3_lsdots -f python tools/prof_gmres.py C3 14 smooth > /dev/null 2>&1
$NCU -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/ncu/c4_persistent -f python tools/prof_apply.py --config C4 --iters 8 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/ncu/bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-gmres > /dev/null 2>&1
ls -la gpurun_out/ncu
