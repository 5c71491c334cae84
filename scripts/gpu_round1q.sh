mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/prof_spmm.py --steps 3 --kernel spmv > gpurun_out/prof_qv.log 2>&1; cat gpurun_out/prof_qv.log
for m in 3 4; do SPD_SDDMM_MINB=$m timeout 900 python scripts/prof_spmm.py --steps 3 --kernel sddmm > gpurun_out/prof_sd$m.log 2>&1; echo "sddmm minb $m exit $?"; cat gpurun_out/prof_sd$m.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sddmm_nz" -s 1 -c 1 -o gpurun_out/prof_sddmm_nz python scripts/prof_spmm.py --steps 2 --kernel sddmm > gpurun_out/ncu_sddmm.log 2>&1; echo "ncu exit $?"
