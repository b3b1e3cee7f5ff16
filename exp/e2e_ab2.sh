# c4 e2e variance: current vs r02g library, alternating, 3 rounds
L=paper_2511_00870_b200
for rep in a b c; do for v in "new:PNPULA_X=0" "old:PNPULA_LIB=$L/libpnpula_old.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --workload c4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e3_$n.json 2>gpurun_out/e3_$n.err
  python -c "import json;d=json.loads(open('gpurun_out/e3_$n.json').read().strip().splitlines()[-1]);e=d['e2e'];print('c4 $n $rep',round(d['value']),'e2e',[round(x) for x in e['reps_mpx_it_s']],'cold',round(e['cold_process']['value']))"
  grep "e2e\]" gpurun_out/e3_$n.err | head -3
done; done
