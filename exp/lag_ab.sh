# layer lag (schedule steps between consecutive layers): 3 (default) vs 4 vs 5, c5
L=paper_2511_00870_b200
PNPULA_LIB=$L/libpnpula_lag4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "denoiser or chain_50_with_cnn" > gpurun_out/lag_tests.log 2>&1; echo "lag4 tests rc=$?"; tail -1 gpurun_out/lag_tests.log
for rep in a b; do for v in "lag3:PNPULA_X=0" "lag4:PNPULA_LIB=$L/libpnpula_lag4.so" "lag5:PNPULA_LIB=$L/libpnpula_lag5.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/lag_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/lag_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done; done
