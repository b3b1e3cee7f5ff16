#!/bin/bash
# kernel timing experiments: same bench, alternative library builds (WL=workload)
WL=${WL:-c2}
for v in "$@"; do
  PNPULA_LIB=exp/lib_$v.so python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$v.log 2>&1
done
