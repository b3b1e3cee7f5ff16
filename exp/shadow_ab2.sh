# shadow-5 diagnosis: ring-4 vs shadow vs shadow plan with ring-4 positions (NOPOS), c5
L=paper_2511_00870_b200
PNPULA_LIB=$L/libpnpula_nopos.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "denoiser or tiled" > gpurun_out/sh_tests2.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/sh_tests2.log
for rep in a b; do for v in "shadow:PNPULA_X=0" "ring4:PNPULA_LIB=$L/libpnpula_ring4.so" "nopos:PNPULA_LIB=$L/libpnpula_nopos.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sh_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sh_$n.json').read().strip().splitlines()[-1]);print('c5 $n $rep',round(d['value']),round(d['ms_per_step'],4),d['kernel_ms_per_step'])"
done; done
