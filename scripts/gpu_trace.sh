# usage: bash scripts/gpu_trace.sh N -- bench with the per-phase trace at N GPUs (N=1: plain python)
N=${1:-1}
mkdir -p gpurun_out
if [ "$N" = "1" ]; then
  timeout 900 python bench.py --steps 10 --warmup 3 --trace --no-cpu-baseline --e2e-steps 1 > gpurun_out/trace_n1.log 2> gpurun_out/trace_n1.err; echo "exit $?"
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 10 --warmup 3 --trace --e2e-steps 1 > gpurun_out/trace_n$N.log 2> gpurun_out/trace_n$N.err; echo "exit $?"
fi
grep trace gpurun_out/trace_n$N.err; tail -1 gpurun_out/trace_n$N.log | cut -c1-400
