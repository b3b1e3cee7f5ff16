# d5 (DDFB) across round-2 commits, same box
L=paper_2511_00870_b200
for v in "r01:PNPULA_LIB=$L/libpnpula_r01.so" "7c84208:PNPULA_LIB=$L/libpnpula_7c84208.so" "cfc6e7d:PNPULA_LIB=$L/libpnpula_cfc6e7d.so" "4a444cd:PNPULA_LIB=$L/libpnpula_4a444cd.so" "4a444cd_nopdl:PNPULA_LIB=$L/libpnpula_4a444cd.so PNPULA_PDL=0" "2db2dac:PNPULA_LIB=$L/libpnpula_2db2dac.so" "now:PNPULA_X=0" "now_nopdl:PNPULA_PDL=0"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload d5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d5b_$n.json 2>gpurun_out/d5b_$n.err
  python -c "import json;d=json.loads(open('gpurun_out/d5b_$n.json').read().strip().splitlines()[-1]);print('d5 $n',round(d['value']),'cnn',round(d['kernel_ms_per_step']['cnn'],4))" || tail -2 gpurun_out/d5b_$n.err
done
