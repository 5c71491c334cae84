mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
for t in 96 192 512; do SPD_SA_T=$t timeout 900 python scripts/bench_configs.py --configs c5 --steps 3 --warmup 1 > gpurun_out/c5_$t.log 2>&1; echo "T=$t"; tail -3 gpurun_out/c5_$t.log; done
