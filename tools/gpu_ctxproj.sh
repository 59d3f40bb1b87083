#!/bin/bash
# projected-context decode: parity + A/B bench against the classic [ctx ; h] operand
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py -q -x 2>&1 | tail -4
KS_CTXPROJ=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_classic.json
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_ctxproj.json
python - <<'PY'
import json
for n in ("classic", "ctxproj"):
    try:
        b = json.load(open(f"gpurun_out/bench_{n}.json"))
        print(n, round(b["value"]), round(b["e2e"]["value"]), b["ms_per_step"], b["roofline"]["all_gemm_launches"])
    except Exception as e:
        print(n, "failed", e)
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_ctxproj.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_ctxproj.csv
