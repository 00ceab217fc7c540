# Round-2 last call on one B200: the full-size golden tests (incl. a freshly
# generated C3 step-7 golden), then two switch checks on the final build.
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -rs > gpurun_out/pytest_fullsize.log 2>&1; echo "pytest fullsize rc $?" >> gpurun_out/ab.txt
tail -8 gpurun_out/pytest_fullsize.log >> gpurun_out/ab.txt
run() {   # tag workload env...
  local tag=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${tag}_$wl.log 2>&1
  echo "== $tag $wl rc $?" >> gpurun_out/ab.txt; python tools/show_bench.py gpurun_out/ab_${tag}_$wl.log 40 >> gpurun_out/ab.txt 2>&1
}
run base C3 A=1
run two7 C3 YY_TH2=7
run utf C3 YY_TH_UTF=1
