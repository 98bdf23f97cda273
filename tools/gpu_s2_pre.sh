for r in 1 2 3; do
python tools/exp_c2.py --tag prefetch=0
TBT_PREFETCH=1 python tools/exp_c2.py --tag prefetch=1
done
