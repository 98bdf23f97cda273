# Round-2 final session (after the C3 changes): GPU suite, smoke, both bench arms, every
# config, launch list, --set full captures (each command ran clean before its ncu pass).
O=gpurun_out/r2d; mkdir -p $O
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader
start=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4; echo "gpu suite $(( $(date +%s) - start )) s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2; echo "smoke rc $?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('$O/bench.json').read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc $?"; head -c 300 $O/bench_reference.json; echo
timeout 1500 python tools/bench_configs.py --configs C1,C2,C3,C4,C5,G48,G40 --out $O/configs.json > $O/configs.log 2>&1; echo "configs rc $?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $O/bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-gmres --no-sharded --no-large > /dev/null 2>&1; echo "launches rc $?"
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:matvecPersistent -s 5 -c 1 -o $O/c2_persistent python tools/prof_apply.py --config C2 --iters 8 > /dev/null 2>&1; echo "c2 rc $?"
$NCU -k regex:"binprodGemm|regLineKernel|corrMulti" -s 12 -c 6 -o $O/c3_apply python tools/prof_apply.py --config C3 --embed smooth --iters 4 > /dev/null 2>&1; echo "c3 rc $?"
ls -la $O
