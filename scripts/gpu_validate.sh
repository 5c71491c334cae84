# Round-end style validation on one B200: GPU parity suite, smoke, bench line
# (with CPU baseline), per-config numbers with full-size oracle checks, and
# the ncu launch list of the bench command.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench1.log 2> gpurun_out/bench1.err; echo "bench exit $?"; tail -1 gpurun_out/bench1.log
timeout 1800 python scripts/bench_configs.py --steps 5 --warmup 2 > gpurun_out/configs.log 2>&1; echo "configs exit $?"; grep '^{' gpurun_out/configs.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1; echo "ncu exit $?"
