mkdir -p gpurun_out
SPD_SA_T=0 timeout 600 compute-sanitizer --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spadd3_hub" > gpurun_out/sanitize_sa.log 2>&1; echo "exit $?"; grep -B2 -A12 "Invalid\|ERROR" gpurun_out/sanitize_sa.log | head -60
