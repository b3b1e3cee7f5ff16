# DDFB residual prefetch by cp.async into shared memory (no register copy): tests, d5 / r5 / c5
timeout 900 python -m pytest tests/test_gpu_ddfb.py tests/test_gpu_rgb.py tests/test_gpu_parity.py -q -x > gpurun_out/da_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/da_tests.log
for rep in a b; do for w in d5 r5 c5; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/da_$w.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/da_$w.json').read().strip().splitlines()[-1]);print('$w $rep',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))"
done; done
