mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
SPD_NZ=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_nz0.log 2>&1; echo "pytest NZ=0 exit $?"; tail -1 gpurun_out/pytest_nz0.log
SPD_DYN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k spmm > gpurun_out/pytest_dyn0.log 2>&1; echo "pytest DYN=0 exit $?"; tail -1 gpurun_out/pytest_dyn0.log
for k in spmm spmv sddmm; do timeout 600 python scripts/prof_spmm.py --steps 4 --kernel $k > gpurun_out/pd.log 2>&1; echo "$k $(tail -1 gpurun_out/pd.log)"; done
