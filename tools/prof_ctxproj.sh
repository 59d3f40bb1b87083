#!/bin/bash
# ncu --set full on the context-projection GEMM and a full-beam alpha-block decoder GEMM
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lstm_gemm_tc" -s 21 -c 4 -o gpurun_out/prof_ctxproj python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_ctxproj.log 2>&1
tail -2 gpurun_out/prof_ctxproj.log
