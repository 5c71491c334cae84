# usage: bash scripts/gpu_mgpu_full.sh N -- parity, all five configs and the bench line at N GPUs
N=${1:-2}
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu$N.log 2>&1; echo "mgpu exit $?"; grep -E "MGPU|Error" gpurun_out/mgpu$N.log | head
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 scripts/mgpu_configs.py > gpurun_out/mconf$N.log 2> gpurun_out/mconf$N.err; echo "mconf exit $?"; grep '^{' gpurun_out/mconf$N.log | cut -c1-330
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --trace > gpurun_out/bench_n$N.log 2> gpurun_out/bench_n$N.err; echo "bench$N exit $?"; grep trace gpurun_out/bench_n$N.err; tail -1 gpurun_out/bench_n$N.log | cut -c1-300
