mkdir -p gpurun_out
SPD_SA_T=0 timeout 900 python -m pytest tests -m gpu -x -q -k spadd3 > gpurun_out/pytest_sa0.log 2>&1; echo "pytest T=0 exit $?"; tail -3 gpurun_out/pytest_sa0.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
for t in 16 64 256; do SPD_SA_T=$t timeout 900 python scripts/bench_configs.py --configs c5 --steps 3 --warmup 1 > gpurun_out/c5_$t.log 2>&1; echo "T=$t"; tail -1 gpurun_out/c5_$t.log; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/bench_configs.py --configs c5 --steps 1 --warmup 0 --no-check > gpurun_out/ncu_c5.log 2>&1; echo "ncu exit $?"
