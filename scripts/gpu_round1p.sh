mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_p.log 2>&1; cat gpurun_out/prof_p.log
timeout 600 python scripts/prof_spmm.py --steps 3 --kernel spmv > gpurun_out/prof_pv.log 2>&1; cat gpurun_out/prof_pv.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_n1.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_n1.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sddmm" -s 1 -c 1 -o gpurun_out/prof_sddmm python scripts/prof_spmm.py --steps 2 --kernel sddmm > gpurun_out/ncu_sddmm.log 2>&1; echo "ncu exit $?"; tail -2 gpurun_out/ncu_sddmm.log
