# Thomas-sweep check: parity subset, then C3 A/B of YY_THOMAS
mkdir -p gpurun_out
: > gpurun_out/rc_th.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heat.py -m gpu -x -q > gpurun_out/pytest_th.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc_th.txt
for cfg in ${TH_CFGS:-"YY_THOMAS=0" "YY_THOMAS=1"}; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_$tag.log 2>&1
  echo "bench $cfg rc $?" >> gpurun_out/rc_th.txt
  echo "== $cfg" >> gpurun_out/ab_th.txt
  python tools/show_bench.py gpurun_out/bench_$tag.log 40 >> gpurun_out/ab_th.txt 2>&1
done
