# GPU check: the GPU tests (optionally a subset), then the default bench line.
mkdir -p gpurun_out
: > gpurun_out/rc.txt
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc.txt
if [ -z "${NO_BENCH:-}" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/rc.txt
fi
