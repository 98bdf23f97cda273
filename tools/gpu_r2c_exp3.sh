# Two-CTA GEMM as default + hoisted correction loads in the cropping line pass: parity and C3 time.
timeout 1500 python -m pytest tests/test_env_paths.py tests/test_gpu_parity.py tests/test_gmres_large.py -m gpu -q -x 2>&1 | tail -3
python tools/prof_apply.py --config C3 --embed smooth --iters 4 | tail -1
python tools/prof_apply.py --config C3 --embed pow2 --iters 4 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"regLineKernel|binprodGemm|corrMulti" -s 24 -c 6 --csv python tools/prof_apply.py --config C3 --embed smooth --iters 4 2>/dev/null | grep -E "regLine|binprod|corrMulti" | awk -F'","' '{print $5, $NF}' | cut -c1-60,100-200
