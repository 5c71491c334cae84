mkdir -p gpurun_out
timeout 900 python scripts/bench_configs.py --configs c5 --steps 3 --warmup 1 > gpurun_out/c5.log 2>&1; tail -1 gpurun_out/c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/bench_configs.py --configs c5 --steps 1 --warmup 0 --no-check > gpurun_out/ncu_c5.log 2>&1; echo "ncu exit $?"
for v in 4 44 43; do SPD_NZ_MINB=$v timeout 900 python scripts/prof_spmm.py --steps 4 > gpurun_out/pf_$v.log 2>&1; echo "minb $v"; tail -1 gpurun_out/pf_$v.log; done
