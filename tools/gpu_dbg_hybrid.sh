#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "hybrid" 2>&1 | grep -E "Error|assert|passed|failed" | head -30
