# PDL on / off, c5 and c2 (bench, 30 steps)
for w in c5 c2 c3; do for v in 1 0 1 0; do
  PNPULA_PDL=$v timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pdl_$w_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pdl_$w_$v.json').read().strip().splitlines()[-1]);print('$w PDL=$v',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done; done
