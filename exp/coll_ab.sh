# A-operand collector reuse for ring-wrap split MMA pairs (PNPULA_COLLECTOR_A build), c5
L=paper_2511_00870_b200
for rep in a b c; do for v in "base:PNPULA_X=0" "coll:PNPULA_LIB=$L/libpnpula_coll.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/co_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/co_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done; done
PNPULA_LIB=$L/libpnpula_coll.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "denoiser or tiled or chain_50_with_cnn" > gpurun_out/co_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/co_tests.log
