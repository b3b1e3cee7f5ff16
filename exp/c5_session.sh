# c5 / c3 / c2: session-start library vs pre-fusion vs now, same box, alternating
L=paper_2511_00870_b200
for rep in a b; do for v in "start:PNPULA_LIB=$L/libpnpula_2db2dac.so" "prefuse:PNPULA_LIB=$L/libpnpula_93f9917.so" "now:PNPULA_X=0"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c3; do
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cs_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/cs_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4),'upd',round(d['kernel_ms_per_step']['update'],4))"
  done
done; done
