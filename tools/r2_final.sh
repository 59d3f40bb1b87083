#!/bin/bash
# Round-2 evidence on one B200: GPU tests, smoke, every bench workload (our arm and
# the reference arm), per-workload GEMM DRAM traffic, the cfg2 launch list.
mkdir -p gpurun_out/f
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/f/pytest_gpu.txt; cat gpurun_out/f/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 > gpurun_out/f/smoke.txt; cat gpurun_out/f/smoke.txt
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/f/bench_cfg2.json
for w in cfg1 cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/f/bench_$w.json
done
timeout 600 python bench.py --precision bf16 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/f/bench_cfg2_bf16.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/f/bench_reference.json
timeout 600 python bench.py --workload cfg4 --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/f/bench_cfg4_reference.json
for f in gpurun_out/f/bench_*.json; do echo "$f: $(head -c 160 $f)"; done
timeout 2400 python tools/measure_traffic.py cfg2:f16x3 cfg2:bf16 cfg1:f16x3 cfg5:f16x3 cfg3:f16x3 2>&1 | tail -6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/f/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/f/launches_cfg2.csv > gpurun_out/f/launches_cfg2_summary.txt; head -12 gpurun_out/f/launches_cfg2_summary.txt
python tools/gemm_launches.py cfg2 > gpurun_out/f/gemm_cfg2.txt 2>&1; tail -1 gpurun_out/f/gemm_cfg2.txt
