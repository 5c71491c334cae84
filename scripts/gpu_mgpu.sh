# usage: bash scripts/gpu_mgpu.sh N  -- multi-GPU parity + bench at N GPUs
N=${1:-2}
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu$N.log 2>&1; echo "mgpu exit $?"; grep -E "mgpu|MGPU|Error|error" gpurun_out/mgpu$N.log | head -30
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.log 2>&1; echo "bench$N exit $?"; tail -1 gpurun_out/bench_n$N.log
