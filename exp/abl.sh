# CNN ablations (timing only, results garbage): per-launch durations of the two c5 chunks
L=paper_2511_00870_b200
for n in ring4 abl1 abl2 abl4 abl6; do
  PNPULA_LIB=$L/libpnpula_$n.so timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:cnn_chunk -c 8 --csv --log-file gpurun_out/abl_$n.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$n rc=$?"
done
