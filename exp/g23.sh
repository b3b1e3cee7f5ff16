cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_tv.py tests/test_gpu_parity.py tests/test_gpu_poisson.py -x -q 2>&1 | tail -3; echo tests-done
for r in 1 2; do for v in base tvm2; do for wl in t5 c5; do
PNPULA_LIB=exp/lib_$v.so timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v$r$wl.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab_$v$r$wl.json').read().strip().splitlines()[-1]); print('$v$r $wl', round(d['value']), d['kernel_ms_per_step'])"
done; done; done
