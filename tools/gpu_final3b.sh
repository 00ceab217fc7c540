# Round-2 closing run, second part (final build): the remaining bench lines
mkdir -p gpurun_out
: > gpurun_out/rc_f3b.txt
B="timeout 900 python bench.py"
$B --steps 100 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_100.log 2>&1; echo "c3 100 rc $?" >> gpurun_out/rc_f3b.txt
$B --advection imex --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_imex.log 2>&1; echo "imex rc $?" >> gpurun_out/rc_f3b.txt
$B --workload C5 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_50.log 2>&1; echo "c5 50 rc $?" >> gpurun_out/rc_f3b.txt
$B --workload C2 --steps 20 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc $?" >> gpurun_out/rc_f3b.txt
$B --workload C2 --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_200.log 2>&1; echo "c2 200 rc $?" >> gpurun_out/rc_f3b.txt
$B --workload C1 --steps 10 > gpurun_out/bench_c1.log 2>&1; echo "c1 rc $?" >> gpurun_out/rc_f3b.txt
timeout 600 python tools/c4_bench.py > gpurun_out/c4.log 2>&1; echo "c4 rc $?" >> gpurun_out/rc_f3b.txt
echo "done" >> gpurun_out/rc_f3b.txt
