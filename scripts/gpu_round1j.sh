mkdir -p gpurun_out
for m in 1 4 5 6; do SPD_NZ_MINB=$m timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_minb$m.log 2>&1; echo "minb $m exit $?"; cat gpurun_out/prof_minb$m.log; done
SPD_NZ_MINB=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmm" > gpurun_out/pytest_minb4.log 2>&1; echo "pytest minb4 exit $?"; tail -1 gpurun_out/pytest_minb4.log
