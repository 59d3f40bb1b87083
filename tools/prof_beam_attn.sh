#!/bin/bash
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"beam_step_t|attention_cta_t" -s 20 -c 2 -o gpurun_out/prof_beam_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_beam_attn.log 2>&1
tail -1 gpurun_out/prof_beam_attn.log
