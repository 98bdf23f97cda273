for r in 1 2; do
python tools/exp_gmres.py --tag lagged
TBT_GMRES=nolag python tools/exp_gmres.py --tag nolag
done
TBT_CTATRACE=1 python tools/cta_trace_gmres.py
python tools/exp_gmres.py --config C4 --iters 50 --tag C4
