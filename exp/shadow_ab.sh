# shadow-5 accumulator layout (default build) vs ring-4 (PNPULA_SHADOW=0) vs shadow with >= 2 im2col slots, c5 / c2
L=paper_2511_00870_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiling_fuzz.py tests/test_gpu_c3_chain.py -q -x > gpurun_out/sh_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sh_tests.log
for rep in a b; do for v in "shadow:PNPULA_X=0" "ring4:PNPULA_LIB=$L/libpnpula_ring4.so" "sh2:PNPULA_LIB=$L/libpnpula_sh2.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sh_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sh_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done; done
for v in "shadow:PNPULA_X=0" "ring4:PNPULA_LIB=$L/libpnpula_ring4.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload c2 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sh2_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sh2_$n.json').read().strip().splitlines()[-1]);print('c2 $n',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done
