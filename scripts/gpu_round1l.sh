mkdir -p gpurun_out
SPD_NZ_MINB=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmm" > gpurun_out/pytest_l.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_l.log
SPD_HOT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmm" > gpurun_out/pytest_lh.log 2>&1; echo "pytest hot exit $?"; tail -1 gpurun_out/pytest_lh.log
for m in 1 4; do SPD_NZ_MINB=$m timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_m$m.log 2>&1; echo "minb $m exit $?"; cat gpurun_out/prof_m$m.log; done
SPD_HOT=1 timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_hot.log 2>&1; echo "hot exit $?"; cat gpurun_out/prof_hot.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm32_nz" -s 1 -c 1 -o gpurun_out/prof_spmm_l python scripts/prof_spmm.py --steps 2 > gpurun_out/ncu_l.log 2>&1; echo "ncu exit $?"
