cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err; tail -c 600 gpurun_out/c5.json
timeout 600 python bench.py --workload r5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r5.json 2> gpurun_out/r5.err; tail -c 600 gpurun_out/r5.json; tail -3 gpurun_out/r5.err
