cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q 2>&1 | tail -2
for r in 1 2; do for v in base relu; do for st in 10 60; do
PNPULA_LIB=exp/lib_$v.so timeout 300 python bench.py --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v$r$st.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab_$v$r$st.json').read().strip().splitlines()[-1]); print('$v$r steps=$st', round(d['value']), d['kernel_ms_per_step'], d['clocks'].get('power_w_max'))"
done; done; done
