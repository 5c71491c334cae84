mkdir -p gpurun_out
for v in 11 13; do SPD_SPMM32_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmm" > gpurun_out/pytest_v$v.log 2>&1; echo "pytest v$v exit $?"; tail -1 gpurun_out/pytest_v$v.log; done
for v in 1 10 11 12 13; do SPD_SPMM32_VARIANT=$v timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_v$v.log 2>&1; echo "variant $v exit $?"; cat gpurun_out/prof_v$v.log; done
