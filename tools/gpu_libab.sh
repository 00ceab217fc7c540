# A/B of alternative builds (YY_LIB) on the C3 (and C5) bench: LIBS="base build/vA ..."
mkdir -p gpurun_out; rm -f gpurun_out/libab.txt
for w in ${WLS:-C3}; do
for v in ${LIBS:-base}; do
  if [ "$v" = base ]; then L=""; else L="YY_LIB=$PWD/$v/libyy.so"; fi
  env $L timeout 600 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/libab_$(basename $v)_$w.log 2>&1
  echo "== $v $w rc $?" >> gpurun_out/libab.txt; python tools/show_bench.py gpurun_out/libab_$(basename $v)_$w.log 40 >> gpurun_out/libab.txt 2>&1
done; done
