for w in d5 r5 p5 t5; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_$w.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02_bench_$w.json').read().strip().splitlines()[-1]);print('$w',round(d['value']),round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['kernel_ms_per_step'].items()})"
done
