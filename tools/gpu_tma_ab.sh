# TMA r/theta sweeps: parity tests, then the C3 bench with YY_TMA=0/1 (twice)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heat.py tests/test_dist.py -x -q > gpurun_out/pytest_tma.log 2>&1
echo "pytest rc $?" > gpurun_out/rc_tma.txt
: > gpurun_out/ab_tma.txt
for v in 0 1 0 1; do
  YY_TMA=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/var.log 2>&1
  echo "== YY_TMA=$v rc $?" >> gpurun_out/ab_tma.txt
  python tools/show_bench.py gpurun_out/var.log 24 >> gpurun_out/ab_tma.txt 2>&1
done
