#!/bin/bash
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
echo "== fused"; timeout 300 python tools/quick_tc.py f16x3 bf16 2>&1 | grep -v Warn | grep -v print | tail -5
echo "== unfused"; KS_FUSE_ATTN=0 timeout 300 python tools/quick_tc.py f16x3 2>&1 | grep -v Warn | grep -v print | tail -3
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_f16x3.json
python -c "import json;b=json.load(open('gpurun_out/bench_f16x3.json'));print('BENCH', b['value'], b['e2e']['value'], b['roofline']['frac'], b['roofline']['gemm_share_of_step'], b['clocks'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
