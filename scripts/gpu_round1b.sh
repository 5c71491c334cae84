mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_plain.log 2>&1; echo "prof plain exit $?"; cat gpurun_out/prof_plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_spmm.py --steps 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_walk -s 1 -c 1 -o gpurun_out/prof_spmm python scripts/prof_spmm.py --steps 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?"; tail -3 gpurun_out/ncu_full.log
