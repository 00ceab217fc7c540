# every GPU test, then the C3 bench A/B (k_line_th on / off) and C5
mkdir -p gpurun_out
: > gpurun_out/rc_full.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc_full.txt
rm -f gpurun_out/ab_th.txt
for cfg in "YY_THOMAS=1" "YY_THOMAS=0"; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$tag.log 2>&1
  echo "bench $cfg rc $?" >> gpurun_out/rc_full.txt
  echo "== $cfg" >> gpurun_out/ab_th.txt
  python tools/show_bench.py gpurun_out/bench_$tag.log 40 >> gpurun_out/ab_th.txt 2>&1
done
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "c5 rc $?" >> gpurun_out/rc_full.txt
