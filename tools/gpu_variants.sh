# A/B of alternative builds of libyy.so (YY_LIB) on the C3 bench line:
#   VARIANTS="build/v_a build/v_b" [OUT=name] [BENCH_ARGS=...] bash tools/gpu_variants.sh
mkdir -p gpurun_out
OUT=gpurun_out/${OUT:-variants}.txt
: > $OUT
for rep in 1 2; do
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then lib=""; else lib="$v/libyy.so"; fi
    YY_LIB=$lib timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/var.log 2>&1
    echo "== $v rep $rep rc $?" >> $OUT
    python tools/show_bench.py gpurun_out/var.log ${NCLS:-12} >> $OUT 2>&1
  done
done
