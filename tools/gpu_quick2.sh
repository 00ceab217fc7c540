# parity subset + C3 and C5 bench lines (kernel classes)
mkdir -p gpurun_out
: > gpurun_out/rc_q2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heat.py -m gpu -x -q > gpurun_out/pytest_q2.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc_q2.txt
rm -f gpurun_out/q2.txt
for w in ${WLS:-C3 C5}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_q2_$w.log 2>&1; echo "bench $w rc $?" >> gpurun_out/rc_q2.txt
  echo "== $w" >> gpurun_out/q2.txt; python tools/show_bench.py gpurun_out/bench_q2_$w.log 40 >> gpurun_out/q2.txt 2>&1
done
