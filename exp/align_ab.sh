# ring alignment A/B (PNPULA_RING_ALIGN build switch), c5 + c2
L=paper_2511_00870_b200
for rep in a b; do
  for v in "align:PNPULA_X=0" "noalign:PNPULA_LIB=$L/libpnpula_noalign.so"; do
    n=${v%%:*}; e=${v#*:}
    env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/al_$n.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/al_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
  done
done
