# A/B of an env switch on the C3 bench (no e2e / cpu baseline), plus quick parity tests.
# usage: VAR=YY_PIPE A=0 B=1 bash tools/gpu_ab.sh
mkdir -p gpurun_out
: > gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc.txt
for v in ${A:-0} ${B:-1} ${A:-0} ${B:-1}; do
  env ${VAR:-YY_PIPE}=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_${VAR:-YY_PIPE}_$v.log 2>&1
  echo "bench $v rc $?" >> gpurun_out/rc.txt
  python tools/show_bench.py gpurun_out/bench_${VAR:-YY_PIPE}_$v.log >> gpurun_out/ab.txt 2>&1
done
