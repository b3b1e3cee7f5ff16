# update kernel: default (2 CTAs, operands loaded early) vs late loads vs late loads + 3 CTAs/SM; c5 / c4 / c3
L=paper_2511_00870_b200
PNPULA_LIB=$L/libpnpula_ll3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or tiled" > gpurun_out/u3_tests.log 2>&1; echo "ll3 tests rc=$?"; tail -1 gpurun_out/u3_tests.log
for rep in a b; do for v in "base:PNPULA_X=0" "ll:PNPULA_LIB=$L/libpnpula_ll.so" "ll3:PNPULA_LIB=$L/libpnpula_ll3.so"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c4; do
  st=50; [ $w = c5 ] && st=30
  env $e timeout 300 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/u3_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/u3_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4),'upd',round(d['kernel_ms_per_step']['update'],4),round(d['roofline_update']['frac'],3))"
  done
done; done
