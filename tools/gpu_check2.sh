#!/bin/bash
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
echo "== units 64"; timeout 300 python tools/quick_tc.py f16x3 bf16 fp32 2>&1 | grep -v Warn | grep -v print | tail -9
echo "== units 32"; KS_TC_UNITS=32 timeout 300 python tools/quick_tc.py f16x3 bf16 2>&1 | grep -v Warn | grep -v print | tail -6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
