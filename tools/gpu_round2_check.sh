mkdir -p gpurun_out
: > gpurun_out/rc13.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc13.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "c3 rc $?" >> gpurun_out/rc13.txt
timeout 600 python bench.py --advection imex --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_imex.log 2>&1; echo "imex rc $?" >> gpurun_out/rc13.txt
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc $?" >> gpurun_out/rc13.txt
