# C3 GMRES (162 lockstep columns, smooth embedding): launch list of iterations ~20-30, full captures of the LS kernels.
O=gpurun_out/r2c; mkdir -p $O
python tools/prof_gmres.py C3 30 smooth | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c3_gmres_launches.csv python tools/prof_gmres.py C3 30 smooth > /dev/null 2>&1; echo "launches rc $?"
python tools/launch_summary.py $O/c3_gmres_launches.csv | tail -25
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:"lsColsDots|lsColsUpdate|lsColsFinish|lsColsSolve|colReduce" -s 125 -c 6 -o $O/c3_ls python tools/prof_gmres.py C3 30 smooth > /dev/null 2>&1; echo "ls rc $?"
