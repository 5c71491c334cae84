mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
SPD_SA_T=0 timeout 900 python -m pytest tests -m gpu -x -q -k spadd3 > gpurun_out/pytest_sa0.log 2>&1; echo "pytest T=0 exit $?"; tail -1 gpurun_out/pytest_sa0.log
for t in 8 16 32; do SPD_SA_T=$t timeout 900 python scripts/bench_configs.py --configs c5 --steps 3 --warmup 1 > gpurun_out/c5_$t.log 2>&1; echo "T=$t $(tail -1 gpurun_out/c5_$t.log | cut -c1-250)"; done
timeout 600 python scripts/prof_spmm.py --steps 4 > gpurun_out/pd.log 2>&1; tail -1 gpurun_out/pd.log
