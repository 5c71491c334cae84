mkdir -p gpurun_out
nvidia-smi topo -m | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu2.log 2>&1; echo "mgpu exit $?"; grep -E "mgpu|MGPU|Error|error" gpurun_out/mgpu2.log | head -20
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.log 2>&1; echo "bench2 exit $?"; tail -1 gpurun_out/bench_n2.log
