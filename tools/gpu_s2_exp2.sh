# Interleaved A/B: cooperative vs plain launch, PDL vs cached graph.
for r in 1 2 3; do
  python tools/exp_c2.py --tag default
  TBT_COOP=0 python tools/exp_c2.py --tag coop=0
  TBT_PDL=0 python tools/exp_c2.py --tag pdl=0
  TBT_PDL=0 TBT_COOP=0 python tools/exp_c2.py --tag pdl=0,coop=0
done
TBT_CTATRACE=1 TBT_COOP=0 timeout 300 python tools/cta_trace.py --config C2 | head -14
