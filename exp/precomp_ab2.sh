L=paper_2511_00870_b200
for rep in a b; do for v in "pre0:PNPULA_LIB=$L/libpnpula_pre0.so" "base:PNPULA_LIB=$L/libpnpula_base.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pc0_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pc0_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done; done
