python tools/exp_gmres.py --tag lagged
TBT_PDL=0 python tools/exp_gmres.py --tag lagged,pdl=0
TBT_GMRES=nolag python tools/exp_gmres.py --tag nolag
TBT_GMRES=nolag TBT_PDL=0 python tools/exp_gmres.py --tag nolag,pdl=0
TBT_CTATRACE=1 python tools/cta_trace_gmres.py
TBT_CTATRACE=1 TBT_GMRES=nolag python tools/cta_trace_gmres.py
