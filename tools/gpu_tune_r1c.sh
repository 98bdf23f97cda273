# L2 prefetch of the spectrum during the forward transforms at C4 / C5 (TBT_DEV_L2="MB,at").
mkdir -p gpurun_out
for v in "0,0" "64,1" "96,1" "96,0" "0,0"; do
  echo "== C4 TBT_DEV_L2=$v"
  TBT_DEV_L2=$v timeout 300 python tools/prof_phases.py --config C4 --n 30 2>&1 | tail -6
done
for v in "0,0" "96,1"; do
  echo "== C5 TBT_DEV_L2=$v"
  TBT_DEV_L2=$v timeout 600 python tools/prof_phases.py --config C5 --n 10 2>&1 | tail -6
done
