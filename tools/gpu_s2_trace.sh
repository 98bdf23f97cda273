# Per-CTA timeline of back-to-back C2 / C4 applies and the C2 GMRES LS split.
TBT_CTATRACE=1 timeout 300 python tools/cta_trace.py --config C2
TBT_CTATRACE=1 timeout 300 python tools/cta_trace.py --config C4 --rounds 5
TBT_LSPROF=1 timeout 300 python tools/prof_gmres.py C2 200
