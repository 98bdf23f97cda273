for r in 0 2 3 0 2 3; do TBT_RING=$r python tools/exp_c2.py --config C4 --n 300 --tag ring=$r; done
for r in 0 1 0 1; do TBT_RING=$r python tools/exp_c2.py --config C5 --n 30 --tag ring=$r; done
