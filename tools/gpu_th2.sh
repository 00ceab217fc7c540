# Round-2 (late) A/B on one B200: the two-way k_line_th (YY_TH2 bit mask: 1 plain r,
# 2 plain theta, 4 final) against the one-warp tiles; GPU tests on the new build first.
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab.txt
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/ab.txt
run() {   # tag workload env...
  local tag=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $wl --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${tag}_$wl.log 2>&1
  echo "== $tag $wl rc $?" >> gpurun_out/ab.txt; python tools/show_bench.py gpurun_out/ab_${tag}_$wl.log 40 >> gpurun_out/ab.txt 2>&1
}
for rep in 1 2; do
  run two7 C3 YY_TH2=7
  run two0 C3 YY_TH2=0
done
run two3 C3 YY_TH2=3
run two4 C3 YY_TH2=4
run two7utf C3 YY_TH2=7 YY_TH_UTF=1
run two7 C5 YY_TH2=7
run two0 C5 YY_TH2=0
