# Round-2 closing evidence on one B200: smoke, every GPU test, the bench lines of
# every BASELINE workload (incl. their full BASELINE lengths), the reference arm,
# the C4 kernel-only sweeps.  Outputs under gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
: > gpurun_out/rc_final.txt
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/rc_final.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc_final.txt
B="timeout 900 python bench.py"
$B > gpurun_out/bench_c3.log 2>&1; echo "c3 rc $?" >> gpurun_out/rc_final.txt
$B --steps 100 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_100.log 2>&1; echo "c3 100 rc $?" >> gpurun_out/rc_final.txt
$B --workload C5 --steps 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc $?" >> gpurun_out/rc_final.txt
$B --workload C5 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_50.log 2>&1; echo "c5 50 rc $?" >> gpurun_out/rc_final.txt
$B --workload C5 --steps 5 --fixed-iters 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_k10.log 2>&1; echo "c5 k10 rc $?" >> gpurun_out/rc_final.txt
$B --workload C2 --steps 20 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc $?" >> gpurun_out/rc_final.txt
$B --workload C2 --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_200.log 2>&1; echo "c2 200 rc $?" >> gpurun_out/rc_final.txt
$B --workload C1 --steps 10 > gpurun_out/bench_c1.log 2>&1; echo "c1 rc $?" >> gpurun_out/rc_final.txt
timeout 600 python tools/c4_bench.py > gpurun_out/c4.log 2>&1; echo "c4 rc $?" >> gpurun_out/rc_final.txt
$B --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3.log 2>&1; echo "ref rc $?" >> gpurun_out/rc_final.txt
