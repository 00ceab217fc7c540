# Round-2 late switch checks on the final build (one B200)
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
run() {   # tag workload env...
  local tag=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${tag}_$wl.log 2>&1
  echo "== $tag $wl rc $?" >> gpurun_out/ab.txt; python tools/show_bench.py gpurun_out/ab_${tag}_$wl.log 40 >> gpurun_out/ab.txt 2>&1
}
run base C3 A=1
run gb8 C3 YY_LIB=$PWD/build/gb8/libyy.so
run two7 C3 YY_TH2=7
run utf C3 YY_TH_UTF=1
run base C3 A=2
run gb8 C3 YY_LIB=$PWD/build/gb8/libyy.so
run base C5 A=1
run gb8 C5 YY_LIB=$PWD/build/gb8/libyy.so
