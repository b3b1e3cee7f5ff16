cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --workload p5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/p5_launches.csv python bench.py --workload p5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:z1_sep -s 2 -c 1 -o gpurun_out/prof_z1 -f python bench.py --workload p5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo rc=$?
