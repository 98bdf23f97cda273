for r in 1 2; do
python tools/exp_c2.py --config C4 --n 300 --tag pf
TBT_PFN=0 python tools/exp_c2.py --config C4 --n 300 --tag nopf
done
python tools/exp_c2.py --config C5 --n 40 --tag pf
TBT_PFN=0 python tools/exp_c2.py --config C5 --n 40 --tag nopf
python tools/exp_c2.py --tag C2
