mkdir -p gpurun_out
for cfg in "SPD_SPMV_X=0" "SPD_SPMV_X=1" "SPD_SPMV_X=2" "SPD_SPMV_MINB=4" "SPD_SPMV_X=1 SPD_SPMV_MINB=4"; do
  env $cfg timeout 600 python scripts/prof_spmm.py --steps 4 --kernel spmv > gpurun_out/pd.log 2>&1; echo "[$cfg] $(tail -1 gpurun_out/pd.log)"
done
SPD_SPMV_X=1 SPD_SPMV_MINB=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spmv or spttv" > gpurun_out/pt.log 2>&1; echo "pytest $?"; tail -1 gpurun_out/pt.log
