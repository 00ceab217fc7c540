mkdir -p gpurun_out
for m in 6 8 12; do YY_LINE_MCAP=$m timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_m$m.log 2>&1; done
