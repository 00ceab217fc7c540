# quick experiment: parity tests (PYTEST_K selects; ALL runs everything), short benches
# under each env setting in $VARIANTS ("name:VAR=val+VAR=val ..."), optional ncu of $NCU_K
mkdir -p gpurun_out
: > gpurun_out/rc.txt
if [ -n "${PYTEST_K:-}" ]; then
  if [ "$PYTEST_K" = ALL ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  else timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; fi
  echo "pytest rc $?" >> gpurun_out/rc.txt
fi
for v in ${VARIANTS:-base:}; do
  name=${v%%:*}; envs=${v#*:}
  env ${envs//+/ } timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$name.log 2>&1
  echo "bench $name rc $?" >> gpurun_out/rc.txt
done
if [ -n "${NCU_K:-}" ]; then
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-3000} -c ${NCU_C:-14} -o gpurun_out/prof_try $B > gpurun_out/ncu_try.log 2>&1; echo "ncu rc $?" >> gpurun_out/rc.txt
fi
if [ -n "${NCU_DEM:-}" ]; then   # capture kernels by demangled-name regex (template args included)
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$NCU_DEM" -s ${NCU_S:-0} -c ${NCU_C:-3} -o gpurun_out/prof_dem $B > gpurun_out/ncu_dem.log 2>&1; echo "ncu_dem rc $?" >> gpurun_out/rc.txt
fi
