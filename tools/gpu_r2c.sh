# Round-2 (late) A/B on one B200: GPU tests on the current build, then the C3 /
# C5 bench with and without the theta-pair tiles (YY_PAIR) and the phi-menu
# variant libraries (build/ph1: (64, 6), build/ph2: (128, 3) for 257-384-row lines).
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab.txt
run() {   # tag workload env...
  local tag=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${tag}_$wl.log 2>&1
  echo "== $tag $wl rc $?" >> gpurun_out/ab.txt; python tools/show_bench.py gpurun_out/ab_${tag}_$wl.log 40 >> gpurun_out/ab.txt 2>&1
}
for rep in 1 2; do
  run base C3 A=1
  run nopair C3 YY_PAIR=0
  [ -f build/ph1/libyy.so ] && run ph1 C3 YY_LIB=$PWD/build/ph1/libyy.so
  [ -f build/ph2/libyy.so ] && run ph2 C3 YY_LIB=$PWD/build/ph2/libyy.so
done
run base C5 A=1
run nopair C5 YY_PAIR=0
