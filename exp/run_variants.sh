#!/bin/bash
# kernel timing experiments: same bench, alternative library builds
for v in "$@"; do
  PNPULA_LIB=exp/lib_$v.so python bench.py --workload c2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$v.log 2>&1
done
