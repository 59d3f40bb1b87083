#!/bin/bash
# CTA-pair GEMM: full GPU suite + cfg2 bench + launch list with KS_TC_PAIR=1
export KS_TC_PAIR=1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/gpu_quick.sh
