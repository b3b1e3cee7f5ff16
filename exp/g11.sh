cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:update_sep -s 4 -c 1 -o gpurun_out/prof_update_c5_v4 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_u.log 2>&1; echo "rc=$?"
python bench.py --workload t5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"update_sep|tv_z" -s 4 -c 2 -o gpurun_out/prof_t5 -f python bench.py --workload t5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_t5.log 2>&1; echo "rc=$?"
