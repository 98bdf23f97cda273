for r in 1 2; do
python tools/exp_e2e.py --tag default
TBT_COOP=1 python tools/exp_e2e.py --tag coop=1
TBT_PDL=0 python tools/exp_e2e.py --tag pdl=0
done
