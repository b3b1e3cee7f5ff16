# layers per CNN launch: 4 (default planner) vs 3 vs 2 (PNPULA_MAX_NL), c5 / c3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "denoiser or chain_50_with_cnn" > gpurun_out/mnl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/mnl_tests.log
for rep in a b; do for v in "nl4:PNPULA_X=0" "nl3:PNPULA_MAX_NL=3" "nl2:PNPULA_MAX_NL=2"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c3; do
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mnl_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/mnl_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4),d['roofline']['kernel'])"
  done
done; done
