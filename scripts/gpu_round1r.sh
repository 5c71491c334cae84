mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/prof_c4.py --kernel spmttkrp > gpurun_out/prof_c4m.log 2>&1; cat gpurun_out/prof_c4m.log | tail -1
timeout 600 python scripts/prof_c4.py --kernel spttv > gpurun_out/prof_c4t.log 2>&1; cat gpurun_out/prof_c4t.log | tail -1
for f in 0.5 0.9 1.2; do SPD_HOT_FRAC=$f timeout 900 python scripts/prof_spmm.py --steps 3 --kernel sddmm > gpurun_out/prof_sdf.log 2>&1; echo "sddmm frac $f"; cat gpurun_out/prof_sdf.log; done
