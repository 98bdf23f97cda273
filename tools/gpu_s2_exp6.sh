TBT_CTATRACE=1 python tools/cta_trace_gmres.py
TBT_CTATRACE=1 TBT_GMRES=nolag python tools/cta_trace_gmres.py
