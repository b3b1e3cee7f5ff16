# DDFB launches with the contiguous decomposition (default) vs row blocks, d5; DDFB tests
timeout 900 python -m pytest tests/test_gpu_ddfb.py tests/test_gpu_rgb.py -q -x > gpurun_out/ctd_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ctd_tests.log
for rep in a b; do for v in "contig:PNPULA_X=0" "blocks:PNPULA_CNN_CONTIG=0"; do
  n=${v%%:*}; e=${v#*:}
  for w in d5 r5; do
  env $e timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ctd_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ctd_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
  done
done; done
