# Round-2 (second session) measurement, part 2: C3 register line passes and
# one fused (lagged) C2 GMRES node.
mkdir -p gpurun_out/r2b
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:regLineKernel -s 8 -c 4 -o gpurun_out/r2b/c3_reglines python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1; echo "reglines rc $?"
$NCU -k regex:matvecPersistent -s 20 -c 1 -o gpurun_out/r2b/c2_gmres_node python tools/prof_gmres.py C2 50 > /dev/null 2>&1; echo "gmres node rc $?"
du -sh gpurun_out
