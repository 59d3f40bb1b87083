#!/bin/bash
# round-2 verification on a fresh box: gpu tests, smoke, default bench, bf16, reference arm, launch list
mkdir -p gpurun_out/v
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/v/pytest_gpu.txt
tail -3 gpurun_out/v/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/v/bench_cfg2.json
timeout 600 python bench.py --precision bf16 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/v/bench_cfg2_bf16.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/v/bench_reference.json
for f in gpurun_out/v/bench_*.json; do echo "$f: $(head -c 600 $f)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/v/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/v/launches.csv > gpurun_out/v/launches_summary.txt; head -30 gpurun_out/v/launches_summary.txt
