#!/bin/bash
# ncu --set full of decoder gate-GEMM launches (cfg2, one step): skip the encoder + P GEMMs
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lstm_gemm_tc" -s ${SKIP:-11} -c ${COUNT:-3} -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_gemm.log 2>&1
tail -1 gpurun_out/prof_gemm.log
