#!/bin/bash
# ncu --set full of one decode step's beam_step / attention_pack launches (cfg2)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"beam_step_t" -s 3 -c 1 -o gpurun_out/prof_beam python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_beam.log 2>&1
tail -1 gpurun_out/prof_beam.log
