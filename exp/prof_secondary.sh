# ncu full captures of the dominant kernels of the secondary workloads (d5, t5, p5, r5), one B200
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
for wl in d5 t5 p5 r5; do python bench.py --workload $wl $B > /dev/null 2>&1 || echo "$wl plain failed"; done
ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 4 -c 2 -o gpurun_out/prof_d5 -f python bench.py --workload d5 $B > /dev/null 2>&1; echo "d5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"update_sep|tv_z" -s 4 -c 2 -o gpurun_out/prof_t5 -f python bench.py --workload t5 $B > /dev/null 2>&1; echo "t5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"update_sep|z1_sep" -s 4 -c 2 -o gpurun_out/prof_p5 -f python bench.py --workload p5 $B > /dev/null 2>&1; echo "p5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 4 -c 2 -o gpurun_out/prof_r5 -f python bench.py --workload r5 $B > /dev/null 2>&1; echo "r5 rc=$?"
