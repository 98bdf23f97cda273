# C3 experiments: DADD cost inside a DMMA stream; GEMM variants; line-pass block size.
cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64test.cu -o fp64test && ./fp64test | tail -8; cd ..
for g in 3m 4m nodadd; do echo "GEMM $g"; TBT_GEMM=$g python tools/prof_apply.py --config C3 --embed smooth --iters 4 | tail -1; done
for b in 128 64 32; do echo "REGBLOCK $b"; TBT_REGBLOCK=$b python tools/prof_apply.py --config C3 --embed smooth --iters 4 | tail -1; done
for b in 128 64; do
TBT_REGBLOCK=$b ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"regLineKernel|binprodGemm" -s 20 -c 5 --csv python tools/prof_apply.py --config C3 --embed smooth --iters 4 2>/dev/null | grep -E "regLine|binprod" | awk -F'","' '{print $5, $NF}' | cut -c1-120
done
TBT_GEMM=nodadd ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"binprodGemm" -s 4 -c 1 --csv python tools/prof_apply.py --config C3 --embed smooth --iters 4 2>/dev/null | grep -E "binprod" | awk -F'","' '{print $5, $NF}' | cut -c1-120
