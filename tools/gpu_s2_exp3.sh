python tools/exp_c2.py --tag fixed
python tools/exp_c2.py --config C4 --n 300 --tag fixed
python tools/exp_gmres.py --tag cycle
TBT_GMRES=graph python tools/exp_gmres.py --tag graph
python tools/exp_c2.py --tag fixed
