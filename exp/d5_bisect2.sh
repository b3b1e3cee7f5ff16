# d5 (DDFB) across this session's commits, same box
L=paper_2511_00870_b200
for v in "93f9917:PNPULA_LIB=$L/libpnpula_93f9917.so" "a7daafe:PNPULA_LIB=$L/libpnpula_a7daafe.so" "2bd5161:PNPULA_LIB=$L/libpnpula_2bd5161.so" "a959dbe:PNPULA_LIB=$L/libpnpula_a959dbe.so" "6989619:PNPULA_LIB=$L/libpnpula_6989619.so" "now:PNPULA_X=0"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload d5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d5c_$n.json 2>gpurun_out/d5c_$n.err
  python -c "import json;d=json.loads(open('gpurun_out/d5c_$n.json').read().strip().splitlines()[-1]);print('d5 $n',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))" || tail -2 gpurun_out/d5c_$n.err
done
