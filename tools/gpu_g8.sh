# A/B on one B200: 8-row elimination groups (build/g8, -DYY_TH_G=8) against 16
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
run() {   # tag workload env...
  local tag=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${tag}_$wl.log 2>&1
  echo "== $tag $wl rc $?" >> gpurun_out/ab.txt; python tools/show_bench.py gpurun_out/ab_${tag}_$wl.log 40 >> gpurun_out/ab.txt 2>&1
}
for rep in 1 2; do
  run g16 C3 A=1
  run g8 C3 YY_LIB=$PWD/build/g8/libyy.so
done
run g16 C5 A=1
run g8 C5 YY_LIB=$PWD/build/g8/libyy.so
