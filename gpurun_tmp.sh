mkdir -p gpurun_out/t
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_trainloop.py tests/test_train_dp.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/t/bench_cfg4.json; head -c 300 gpurun_out/t/bench_cfg4.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/t/launches_cfg4.csv python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
