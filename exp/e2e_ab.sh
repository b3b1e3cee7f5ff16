# small-config e2e: current library vs the r02g-commit library (b39f514), same box
L=paper_2511_00870_b200
for rep in a b; do for v in "new:PNPULA_X=0" "old:PNPULA_LIB=$L/libpnpula_old.so"; do
  n=${v%%:*}; e=${v#*:}
  for w in c2 c4; do
  env $e timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e2_${w}_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/e2_${w}_$n.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$w $n $rep',round(d['value']),'e2e',[round(x) for x in e['reps_mpx_it_s']],'cold',round(e['cold_process']['value']))"
  done
done; done
