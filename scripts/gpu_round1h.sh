mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/pytest_gpu.log
timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_nz.log 2>&1; echo "spmm nz exit $?"; cat gpurun_out/prof_nz.log
timeout 600 python scripts/prof_spmm.py --steps 3 --kernel spmv > gpurun_out/prof_nz_spmv.log 2>&1; echo "spmv nz exit $?"; cat gpurun_out/prof_nz_spmv.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm32_nz|k_spmv_nz" -s 1 -c 1 -o gpurun_out/prof_spmm_nz python scripts/prof_spmm.py --steps 2 > gpurun_out/ncu_nz.log 2>&1; echo "ncu exit $?"
