# programmatic dependent launch extended to the update / copy kernels: PNPULA_PDL=1 (default) vs 0
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py tests/test_gpu_tiling_fuzz.py -q -x > gpurun_out/pdl2_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pdl2_tests.log
for rep in a b; do for v in "pdl:PNPULA_X=0" "nopdl:PNPULA_PDL=0"; do
  n=${v%%:*}; e=${v#*:}
  for w in c4 c2 c5; do
  st=50; [ $w = c5 ] && st=30
  env $e timeout 300 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pdl2_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pdl2_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4))"
  done
done; done
