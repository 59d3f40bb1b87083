#!/bin/bash
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for m in 0 1 2; do
KS_ATTN_MODE=$m timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_m$m.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo "== attention mode $m"; python tools/launch_summary.py gpurun_out/launches_m$m.csv
done
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_f16x3.json
python -c "import json;b=json.load(open('gpurun_out/bench_f16x3.json'));print('BENCH', b['value'], b['e2e']['value'], b['roofline']['frac'], b['roofline']['gemm_share_of_step'], b['clocks'])"
