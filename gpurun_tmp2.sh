timeout 900 python -m pytest tests/test_gemm16_gpu.py -q 2>&1 | grep -E 'assert|Error|passed|failed' | head -30
