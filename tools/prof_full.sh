#!/bin/bash
# ncu --set full: a full-beam decoder GEMM, attention_cfg and beam_step launch (position 3)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lstm_gemm_tc|attention_cfg_t|beam_step_t" -s 16 -c 3 -o gpurun_out/prof_r1c python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_r1c.log 2>&1
tail -2 gpurun_out/prof_r1c.log
