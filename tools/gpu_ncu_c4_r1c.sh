mkdir -p gpurun_out/ncu
timeout 300 python tools/prof_apply.py --config C4 --iters 8 > /dev/null 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:matvecPersistent -s 5 -c 1 -o gpurun_out/ncu/r1c_c4_persistent -f python tools/prof_apply.py --config C4 --iters 8 > gpurun_out/ncu/c4.log 2>&1
ls -la gpurun_out/ncu/r1c_c4_persistent.ncu-rep
