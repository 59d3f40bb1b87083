#!/bin/bash
# Round-1 evidence: GPU tests, every bench workload, both reference arms, the
# launch list and ncu --set full captures of the top kernels.
mkdir -p gpurun_out/m
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/m/pytest_gpu.txt
cat gpurun_out/m/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/m/bench_cfg2.json
for w in cfg1 cfg3 cfg5 cfg4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/m/bench_$w.json
done
KS_CTXPROJ=0 timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/m/bench_cfg2_classic.json
timeout 600 python bench.py --precision bf16 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/m/bench_cfg2_bf16.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/m/bench_reference.json
timeout 600 python bench.py --workload cfg4 --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/m/bench_cfg4_reference.json
for f in gpurun_out/m/bench_*.json; do echo "$f: $(head -c 200 $f)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/m/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/m/launches.csv > gpurun_out/m/launches_summary.txt; cat gpurun_out/m/launches_summary.txt
# warm-up step = 15 gate GEMMs: skip them and the 6 encoder launches of the timed step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lstm_gemm_tc" -s 21 -c 4 -o gpurun_out/m/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/m/prof_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"beam_step_t|attention_pack_t" -s 20 -c 4 -o gpurun_out/m/prof_beam_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/m/prof_beam_attn.log 2>&1
tail -n 1 gpurun_out/m/prof_gemm.log; tail -n 1 gpurun_out/m/prof_beam_attn.log
