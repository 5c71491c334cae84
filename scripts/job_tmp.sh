mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
for k in spmm spmv sddmm; do timeout 600 python scripts/prof_spmm.py --steps 4 --kernel $k > gpurun_out/pd.log 2>&1; echo "$k $(tail -1 gpurun_out/pd.log)"; done
timeout 600 python scripts/prof_c4.py --kernel spmttkrp > gpurun_out/pd.log 2>&1; tail -1 gpurun_out/pd.log
timeout 600 python scripts/prof_c4.py --kernel spttv > gpurun_out/pd.log 2>&1; tail -1 gpurun_out/pd.log
timeout 600 python scripts/bench_configs.py --configs c1 > gpurun_out/pd.log 2>&1; tail -1 gpurun_out/pd.log | cut -c1-200
