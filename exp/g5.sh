cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r5_launches.csv python bench.py --workload r5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c5_launches.csv python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python - <<'P'
import csv
for f in ("gpurun_out/r5_launches.csv","gpurun_out/c5_launches.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
    print(f)
    for r in rows[1:][-12:]: print("  ", r[ki][:60], r[vi])
P
