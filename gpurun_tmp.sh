timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python tools/gemm_launches.py cfg2 2>&1 | tail -16
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | head -c 300
