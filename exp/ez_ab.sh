# epilogue early re-zeroing (default) vs late (PNPULA_EARLY_ZERO=0 build), c5 / c2
L=paper_2511_00870_b200
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "denoiser or tiled or chain" > gpurun_out/ez_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ez_tests.log
for rep in a b c; do for v in "early:PNPULA_X=0" "late:PNPULA_LIB=$L/libpnpula_lz.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ez_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ez_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done; done
for v in "early:PNPULA_X=0" "late:PNPULA_LIB=$L/libpnpula_lz.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload c2 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ez2_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ez2_$n.json').read().strip().splitlines()[-1]);print('c2 $n',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done
