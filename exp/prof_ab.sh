# ncu --set full of one CNN evaluation, ring-4 (2 launches) vs W6 (3 launches), c5
PNPULA_WSLOTS=4 ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 6 -c 2 -o gpurun_out/prof_ring4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_ring4.log 2>&1; echo "ring4 rc=$?"
PNPULA_WSLOTS=6 ncu --set full --clock-control none --import-source on -k regex:cnn_chunk -s 9 -c 3 -o gpurun_out/prof_w6 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_w6.log 2>&1; echo "w6 rc=$?"
