mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
for h in 0 1; do SPD_HOT=$h timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_hot$h.log 2>&1; echo "hot $h exit $?"; cat gpurun_out/prof_hot$h.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm32_nz" -s 1 -c 1 -o gpurun_out/prof_spmm_hot python scripts/prof_spmm.py --steps 2 > gpurun_out/ncu_hot.log 2>&1; echo "ncu exit $?"
