# Round deliverables on one B200 (run from the repo root through gpurun); outputs in gpurun_out/
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02j_gputests.log 2>&1; echo "tests rc=$?"
python __graft_entry__.py smoke > gpurun_out/r02j_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/r02j_bench_default.json 2> gpurun_out/r02j_bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/r02j_bench_reference.json 2>&1; echo "ref rc=$?"
for w in c2 c3 c4 c1; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r02j_bench_$w.json 2>/dev/null; echo "$w rc=$?"; done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 6 -c 2 -o gpurun_out/r02j_prof_cnn_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cnn.log 2>&1; echo "cnn rc=$?"
ncu --set full --clock-control none --import-source on -k regex:update_sep -s 6 -c 1 -o gpurun_out/r02j_prof_update_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_upd.log 2>&1; echo "upd rc=$?"
