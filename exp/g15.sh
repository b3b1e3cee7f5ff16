cd $GRAFT_REPO_ROOT
for wl in c5 c5 r5 c4; do
PNPULA_TIME_CREATE=1 timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/wl_$wl.json 2> gpurun_out/wl_$wl.err
python -c "import json; d=json.loads(open('gpurun_out/wl_$wl.json').read().strip().splitlines()[-1]); print('$wl', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"; grep "e2e\|pnpula_create" gpurun_out/wl_$wl.err | tail -10
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
