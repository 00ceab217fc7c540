# quick GPU check: parity tests + a short bench (no ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" > gpurun_out/rc.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/rc.txt
