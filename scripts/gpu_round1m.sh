mkdir -p gpurun_out
for m in 4 83 84; do SPD_NZ_MINB=$m timeout 600 python scripts/prof_spmm.py --steps 3 > gpurun_out/prof_m$m.log 2>&1; echo "minb $m exit $?"; cat gpurun_out/prof_m$m.log; done
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1.log 2>&1; echo "bench exit $?"; tail -2 gpurun_out/bench_r1.log
