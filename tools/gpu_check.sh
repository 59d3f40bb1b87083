#!/bin/bash
# parity (all GPU tests) + quick timing + per-launch device times
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 300 python tools/quick_tc.py f16x3 bf16 fp32 2>&1 | grep -v Warning | tail -12
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
