# per-launch durations (ncu launch list) and full captures of CNN chunk 2 for ring-4 / nopos / shadow
L=paper_2511_00870_b200
for v in "shadow:PNPULA_X=0" "ring4:PNPULA_LIB=$L/libpnpula_ring4.so" "nopos:PNPULA_LIB=$L/libpnpula_nopos.so"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cnn_chunk -c 12 --csv --log-file gpurun_out/shp_launch_$n.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$n list rc=$?"
  env $e timeout 900 ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 7 -c 1 -o gpurun_out/shp_$n -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$n full rc=$?"
done
