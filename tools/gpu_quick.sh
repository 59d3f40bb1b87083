#!/bin/bash
# quick A/B: parity subset + cfg2 bench + GEMM launch times
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_quick.json
python - <<'PY'
import json
b = json.load(open("gpurun_out/bench_quick.json"))
r = b["roofline"]
print("cfg2", round(b["value"]), "e2e", round(b["e2e"]["value"]), "ms", round(b["ms_per_step"], 3),
      "gemm_ms", round(r["all_gemm_launches"]["ms_per_step"], 3), "frac", round(r["frac"], 3),
      "issued", round(r["mma_issued_frac"], 3), "fullbeam", r["full_beam_launch"])
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 45 --csv --log-file gpurun_out/launches_quick.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_quick.csv
