# Round-2 (late) A/B on one B200: the fringe interpolation of p / u beside the T
# solve (YY_DEFER_INTERP, default 1) against the joined form; GPU tests first.
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab.txt
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/ab.txt
run() {   # tag workload env...
  local tag=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${tag}_$wl.log 2>&1
  echo "== $tag $wl rc $?" >> gpurun_out/ab.txt; python tools/show_bench.py gpurun_out/ab_${tag}_$wl.log 4 >> gpurun_out/ab.txt 2>&1
}
for rep in 1 2; do
  run defer C3 YY_DEFER_INTERP=1
  run join C3 YY_DEFER_INTERP=0
done
run defer C5 YY_DEFER_INTERP=1
run join C5 YY_DEFER_INTERP=0
STEPS=20 run defer C2 YY_DEFER_INTERP=1
STEPS=20 run join C2 YY_DEFER_INTERP=0
STEPS=20 run defer C1 YY_DEFER_INTERP=1
STEPS=20 run join C1 YY_DEFER_INTERP=0
