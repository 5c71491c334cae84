mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pack.py tests/test_abi.py -m gpu -x -q > gpurun_out/pytest_pack.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_pack.log
timeout 900 python scripts/bench_pack.py > gpurun_out/bench_pack.log 2>&1; echo "bench_pack exit $?"; tail -3 gpurun_out/bench_pack.log
