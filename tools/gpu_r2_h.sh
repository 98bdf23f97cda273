mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:binprodStream -c 1 -o gpurun_out/r2h_stream python tools/prof_apply.py --config G48 --iters 2 > gpurun_out/r2h.log 2>&1
tail -3 gpurun_out/r2h.log
