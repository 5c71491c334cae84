mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sa_long|k_sa_fill|k_sa_count" -c 4 -o gpurun_out/sa_full python scripts/bench_configs.py --configs c5 --steps 1 --warmup 0 --no-check > gpurun_out/ncu_sa.log 2>&1; echo "ncu exit $?"
