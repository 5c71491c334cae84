mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_plain.log 2>&1; echo "prof plain exit $?"; cat gpurun_out/prof_plain.log
timeout 600 python scripts/prof_spmm.py --steps 3 --kernel spmv > gpurun_out/prof_plain_spmv.log 2>&1; echo "prof spmv exit $?"; cat gpurun_out/prof_plain_spmv.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm32_walk -s 1 -c 1 -o gpurun_out/prof_spmm32 python scripts/prof_spmm.py --steps 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?"; tail -2 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_walk -s 1 -c 1 -o gpurun_out/prof_spmv python scripts/prof_spmm.py --steps 3 --kernel spmv > gpurun_out/ncu_full_spmv.log 2>&1; echo "ncu3 exit $?"; tail -2 gpurun_out/ncu_full_spmv.log
