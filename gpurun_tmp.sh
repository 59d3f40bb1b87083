mkdir -p gpurun_out/e
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/gemm_launches.py cfg2 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/e/bench_cfg2.json; head -c 300 gpurun_out/e/bench_cfg2.json
