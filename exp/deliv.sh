set -x
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 4 -c 2 -o gpurun_out/prof_cnn_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cnn.log 2>&1; echo "cnn rc=$?"
ncu --set full --clock-control none --import-source on -k regex:update_sep -s 4 -c 1 -o gpurun_out/prof_update_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_upd.log 2>&1; echo "upd rc=$?"
