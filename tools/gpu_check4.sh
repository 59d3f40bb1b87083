#!/bin/bash
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
echo "== cfg attention"; timeout 300 python tools/quick_tc.py f16x3 2>&1 | grep -v Warn | grep -v print | tail -2
echo "== row attention"; KS_ATTN_PER_ROW=1 timeout 300 python tools/quick_tc.py f16x3 2>&1 | grep -v Warn | grep -v print | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
KS_ATTN_PER_ROW=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_row.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_row.csv | grep attention
