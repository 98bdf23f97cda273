# After the DMMA correction kernel: every config again, the C3 apply's kernels under ncu --set full,
# C3 GMRES launch list (each ncu pass after the same command ran clean).
O=gpurun_out/r2e; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
timeout 1500 python tools/bench_configs.py --configs C1,C2,C3,C4,C5,G48,G40 --out $O/configs.json > $O/configs.log 2>&1; echo "configs rc $?"
python tools/prof_apply.py --config C3 --embed smooth --iters 4 | tail -1
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:"binprodGemm|regLineKernel|corrDmma" -s 12 -c 6 -o $O/c3_apply python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1; echo "c3 rc $?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c3_gmres_launches.csv python tools/prof_gmres.py C3 30 smooth > /dev/null 2>&1; echo "launches rc $?"
python tools/launch_summary.py $O/c3_gmres_launches.csv | tail -16
