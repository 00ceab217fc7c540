mkdir -p gpurun_out; rm -f gpurun_out/c5ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "chunkings or c1_manu or ragged" > gpurun_out/pytest_c5ab.log 2>&1; echo "pytest rc $?" > gpurun_out/rc_c5ab.txt
for v in ${CFGS:-YY_TMA=1 YY_TMA=0}; do
  env $v timeout 600 python bench.py --workload ${WL:-C5} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_$v.log 2>&1
  echo "== $v" >> gpurun_out/c5ab.txt; python tools/show_bench.py gpurun_out/bench_c5_$v.log 40 >> gpurun_out/c5ab.txt 2>&1
done
