mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pack.py -m gpu -x -q > gpurun_out/pytest_pack.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/pytest_pack.log
