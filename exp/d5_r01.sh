# d5 (DDFB) with the round-1 library vs the current one, same box (the r01 library lacks newer ABI
# hooks: PNPULA_LIB skips the debug symbol)
L=paper_2511_00870_b200
for rep in a b; do for v in "now:PNPULA_X=0" "r01:PNPULA_LIB=$L/libpnpula_r01.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload d5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d5_$n.json 2>gpurun_out/d5_$n.err
  python -c "import json;d=json.loads(open('gpurun_out/d5_$n.json').read().strip().splitlines()[-1]);print('d5 $n $rep',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))" || tail -3 gpurun_out/d5_$n.err
done; done
