# A/B of the CNN accumulator schemes on c5 (run on a GPU box from the repo root):
# PNPULA_WSLOTS=4 ring-4 everywhere (2 launches), 5 = W5 (2 launches), 6 = W6 (3 launches)
for v in 4 6 5 6 4; do
  PNPULA_WSLOTS=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);print('WSLOTS=$v',d['kernel_ms_per_step'],round(d['value']),round(d['ms_per_step'],3))"
done
