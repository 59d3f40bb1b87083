timeout 900 python -m pytest tests/test_api_gpu.py tests/test_gemm16_gpu.py tests/test_forward_gpu.py -q 2>&1 | tail -4
