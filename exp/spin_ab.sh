# mbarrier waits: try_wait with a suspend-time hint (default) vs plain spinning (PNPULA_POLL_HINT=0), c5 / c2
L=paper_2511_00870_b200
for rep in a b c; do for v in "hint:PNPULA_X=0" "spin:PNPULA_LIB=$L/libpnpula_spin.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sp_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done; done
for v in "hint:PNPULA_X=0" "spin:PNPULA_LIB=$L/libpnpula_spin.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload c2 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp2_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sp2_$n.json').read().strip().splitlines()[-1]);print('c2 $n',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done
