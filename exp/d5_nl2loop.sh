timeout 600 python -m pytest tests/test_gpu_ddfb.py tests/test_gpu_cnn_decomposition.py -q -x > gpurun_out/dl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/dl_tests.log
for rep in a b; do for w in d5 c5; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dl_$w.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/dl_$w.json').read().strip().splitlines()[-1]);print('$w $rep',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done; done
