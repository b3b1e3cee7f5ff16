# contiguous CNN work ranges per CTA (default) vs row-block units (PNPULA_CNN_CONTIG=0)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiling_fuzz.py tests/test_gpu_c3_chain.py tests/test_gpu_fused_update.py tests/test_gpu_fullsize.py -q -x > gpurun_out/ct_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ct_tests.log
for rep in a b c; do for v in "contig:PNPULA_X=0" "blocks:PNPULA_CNN_CONTIG=0"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c3; do
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ct_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ct_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
  done
done; done
