mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
for v in 1 2 3 4; do SPD_SPMM32_VARIANT=$v timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_v$v.log 2>&1; echo "variant $v exit $?"; cat gpurun_out/prof_v$v.log; done
