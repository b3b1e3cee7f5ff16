# update kernel: incremental block coordinates + interior fast path for the residual (default) vs previous library
L=paper_2511_00870_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiling_fuzz.py tests/test_gpu_fused_update.py -q -x > gpurun_out/um_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/um_tests.log
for rep in a b c; do for v in "new:PNPULA_X=0" "base:PNPULA_LIB=$L/libpnpula_base.so"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c4; do
  st=50; [ $w = c5 ] && st=30
  env $e timeout 300 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/um_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/um_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4),'upd',round(d['kernel_ms_per_step']['update'],4),round(d['roofline_update']['frac'],3))"
  done
done; done
