# A/B of the C2 persistent kernel knobs (back-to-back time + phase split).
for P in 0 1 2; do TBT_PREFETCH=$P python tools/exp_c2.py --tag prefetch=$P; done
TBT_PDL=0 python tools/exp_c2.py --tag pdl=0
python tools/exp_c2.py --config C4 --n 300 --tag default
