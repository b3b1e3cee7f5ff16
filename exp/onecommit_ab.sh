# one tcgen05.commit per fill (epilogue waits on the input ring's empty barrier; default) vs two
L=paper_2511_00870_b200
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiling_fuzz.py tests/test_gpu_c3_chain.py tests/test_gpu_ddfb.py tests/test_gpu_cnn_decomposition.py tests/test_gpu_fused_update.py tests/test_gpu_rgb.py -q -x > gpurun_out/oc_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/oc_tests.log
for rep in a b c; do for v in "one:PNPULA_X=0" "two:PNPULA_LIB=$L/libpnpula_2c.so"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c3; do
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/oc_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/oc_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
  done
done; done
for v in "one:PNPULA_X=0" "two:PNPULA_LIB=$L/libpnpula_2c.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload c2 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/oc2_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/oc2_$n.json').read().strip().splitlines()[-1]);print('c2 $n',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done
