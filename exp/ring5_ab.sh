# epilogue-fed input rings of 5 slots (PNPULA_RING_ACT=5) vs 4, with the contiguous decomposition; c5 / c3
L=paper_2511_00870_b200
PNPULA_LIB=$L/libpnpula_ring5.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "denoiser or chain_50_with_cnn" > gpurun_out/r5_tests.log 2>&1; echo "ring5 tests rc=$?"; tail -1 gpurun_out/r5_tests.log
for rep in a b c; do for v in "ring4:PNPULA_X=0" "ring5:PNPULA_LIB=$L/libpnpula_ring5.so"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c3; do
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r5_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
  done
done; done
