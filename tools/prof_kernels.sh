#!/bin/bash
# one ncu --set full capture of each hot kernel (1 GPU), plus a units=64 timing
set -x
KS_TC_UNITS=64 timeout 300 python tools/quick_tc.py f16x3 bf16 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"beam_step|attention_pack|lstm_gemm_tc|uatt" -s 20 -c 4 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_r1.log 2>&1
tail -3 gpurun_out/prof_r1.log
