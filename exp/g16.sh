cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ddfb.py tests/test_gpu_graphs.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15
for v in ddfb2 ddfb3; do
PNPULA_LIB=exp/lib_$v.so timeout 300 python bench.py --workload d5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v d5', round(d['value']), d['kernel_ms_per_step'], d['roofline']['frac'])"
done
