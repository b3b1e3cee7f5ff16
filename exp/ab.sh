cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3 4; do for v in old new; do
PNPULA_LIB=exp/lib_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v$r.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab_$v$r.json').read().strip().splitlines()[-1]); print('$v$r', round(d['value']), d['kernel_ms_per_step'])"
done; done
