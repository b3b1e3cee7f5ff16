# A/B of CNN kernel builds on c5 (run on a GPU box from the repo root); variant libraries built
# here with build.build(out=..., defines=[...]) and selected with PNPULA_LIB
run() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$1.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_$1.json').read().strip().splitlines()[-1]);print('$1',d['kernel_ms_per_step'],round(d['value']),round(d['ms_per_step'],3))"
}
L=paper_2511_00870_b200
for rep in a b; do
  run base_$rep PNPULA_X=0
  run r1_$rep PNPULA_LIB=$L/libpnpula_r1.so
  run poll32_$rep PNPULA_LIB=$L/libpnpula_poll32.so
  run cvt_$rep PNPULA_LIB=$L/libpnpula_cvt.so
  run both_$rep PNPULA_LIB=$L/libpnpula_both.so
done
