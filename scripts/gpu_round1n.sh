mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_n1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch exit $?"
timeout 2400 python scripts/bench_configs.py --steps 5 --warmup 2 > gpurun_out/configs.log 2>&1; echo "configs exit $?"; cat gpurun_out/configs.log | tail -8
