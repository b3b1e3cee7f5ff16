# full round-end validation on one B200: smoke, deliverables (exp/deliv.sh), every bench workload
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 bash exp/deliv.sh 2>&1 | grep "rc="
for wl in c1 c2 c3 c4 p5 t5 d5 r5; do
timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/wl_$wl.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/wl_$wl.json').read().strip().splitlines()[-1]); print('$wl', round(d['value'],1), round(d['ms_per_step'],4), d['kernel_ms_per_step'], 'e2e', round(d['e2e']['value'],1), 'roof', round(d['roofline']['frac'],3), round(d['roofline_update']['frac'] or 0,3))"
done
