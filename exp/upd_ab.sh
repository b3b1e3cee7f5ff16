# update kernel: 2 vs 3 CTAs per SM (PNPULA_UPD_CTAS build switch), c5 / c4 / t5
L=paper_2511_00870_b200
for w in c5 c4 t5; do for v in "upd2:PNPULA_X=0" "upd3:PNPULA_LIB=$L/libpnpula_upd3.so" "upd2b:PNPULA_X=0" "upd3b:PNPULA_LIB=$L/libpnpula_upd3.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/u_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/u_$n.json').read().strip().splitlines()[-1]);print('$w $n',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'],round(d['roofline_update']['frac'],3))"
done; done
PNPULA_LIB=$L/libpnpula_upd3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "chain_50 or one_iteration" > gpurun_out/u_tests.log 2>&1; echo "tests rc=$?"
