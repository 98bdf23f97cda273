for r in 1 2; do
python tools/exp_gmres.py --tag cycle
TBT_GMRES=graph python tools/exp_gmres.py --tag graph
python tools/exp_c2.py --tag plain+pdl
TBT_COOP=1 python tools/exp_c2.py --tag coop=1
done
python tools/exp_gmres.py --config C4 --iters 50 --tag cycle
TBT_GMRES=graph python tools/exp_gmres.py --config C4 --iters 50 --tag graph
