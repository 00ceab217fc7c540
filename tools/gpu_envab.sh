# A/B of env settings on a bench workload: CFGS="A=1 A=0" WL=C5
mkdir -p gpurun_out; rm -f gpurun_out/envab.txt
for v in ${CFGS}; do
  env $v timeout 600 python bench.py --workload ${WL:-C3} --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/envab_$v.log 2>&1
  echo "== $v rc $?" >> gpurun_out/envab.txt; python tools/show_bench.py gpurun_out/envab_$v.log 40 >> gpurun_out/envab.txt 2>&1
done
