# fused update (PNPULA_FUSE=1) vs unfused (PNPULA_FUSE=0): tests, then c5 / c3 / c2 bench A/B
timeout 900 python -m pytest tests/test_gpu_fused_update.py -q -x > gpurun_out/fu_tests.log 2>&1; echo "fused tests rc=$?"; tail -3 gpurun_out/fu_tests.log
for rep in a b; do for v in "fused:PNPULA_FUSE=1" "unfused:PNPULA_FUSE=0"; do
  n=${v%%:*}; e=${v#*:}
  for w in c5 c3; do
  env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fu_${w}_$n.json 2>gpurun_out/fu_${w}_$n.err
  python -c "import json;d=json.loads(open('gpurun_out/fu_${w}_$n.json').read().strip().splitlines()[-1]);print('$w $n $rep',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
  done
done; done
for v in "fused:PNPULA_FUSE=1" "unfused:PNPULA_FUSE=0"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload c2 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fu_c2_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/fu_c2_$n.json').read().strip().splitlines()[-1]);print('c2 $n',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done
