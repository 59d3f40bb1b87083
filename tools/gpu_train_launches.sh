timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', d['value'], d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg4.csv | head -30
