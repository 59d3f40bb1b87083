#!/bin/bash
# every BASELINE workload on one GPU (+ the reference arm of the headline)
for w in cfg2 cfg3 cfg5 cfg1; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_$w.json
  echo "$w: $(python -c "import json;b=json.load(open('gpurun_out/bench_$w.json'));print(round(b['value']), round(b['e2e']['value']), round(b['roofline']['frac'],3), (b['cpu_baseline'] or {}).get('value'))")"
done
timeout 600 python bench.py --workload cfg2 --steps 10 --warmup 3 --precision bf16 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_cfg2_bf16.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_reference.json
cat gpurun_out/bench_reference.json
