# Round-2 (second half) evidence on one B200 after the one-line-per-thread sweeps:
# smoke, every GPU test, the bench lines of every BASELINE workload (incl. their
# full BASELINE lengths), the reference arm, C4 kernel-only, the ncu launch list
# and one `ncu --set full` capture of a whole Schwarz iteration's hot kernels.
mkdir -p gpurun_out
: > gpurun_out/rc_2b.txt
nvidia-smi > gpurun_out/smi.txt 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/rc_2b.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc_2b.txt
B="timeout 900 python bench.py"
$B > gpurun_out/bench_c3.log 2>&1; echo "c3 rc $?" >> gpurun_out/rc_2b.txt
$B --steps 100 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_100.log 2>&1; echo "c3 100 rc $?" >> gpurun_out/rc_2b.txt
$B --advection imex --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_imex.log 2>&1; echo "imex rc $?" >> gpurun_out/rc_2b.txt
$B --workload C5 --steps 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc $?" >> gpurun_out/rc_2b.txt
$B --workload C5 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_50.log 2>&1; echo "c5 50 rc $?" >> gpurun_out/rc_2b.txt
$B --workload C5 --steps 5 --fixed-iters 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_k10.log 2>&1; echo "c5 k10 rc $?" >> gpurun_out/rc_2b.txt
$B --workload C2 --steps 20 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc $?" >> gpurun_out/rc_2b.txt
$B --workload C2 --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_200.log 2>&1; echo "c2 200 rc $?" >> gpurun_out/rc_2b.txt
$B --workload C1 --steps 10 > gpurun_out/bench_c1.log 2>&1; echo "c1 rc $?" >> gpurun_out/rc_2b.txt
timeout 600 python tools/c4_bench.py > gpurun_out/c4.log 2>&1; echo "c4 rc $?" >> gpurun_out/rc_2b.txt
$B --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3.log 2>&1; echo "ref rc $?" >> gpurun_out/rc_2b.txt
# ncu (a graph with a conditional node is not profiled kernel by kernel: one plain
# graph per Schwarz iteration, the same kernels)
export YY_GRAPH=1
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B1 > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 3000 -c 2500 --csv --log-file gpurun_out/launches.csv $B1 > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc $?" >> gpurun_out/rc_2b.txt
python tools/ncu_launches.py gpurun_out/launches.csv > gpurun_out/launches.md 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_line|k_resid|k_pres|k_interp" -s 3000 -c 40 -f -o /tmp/prof_iter $B1 > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc $?" >> gpurun_out/rc_2b.txt
python tools/ncu_full_summary.py /tmp/prof_iter.ncu-rep > gpurun_out/ncu_full.md 2>&1
python tools/ncu_traffic.py /tmp/prof_iter.ncu-rep r02b > gpurun_out/traffic.json 2>&1
for i in $(seq 0 39); do python tools/ncu_opcodes.py /tmp/prof_iter.ncu-rep $i 2>/dev/null | head -3; done > gpurun_out/ncu_opcodes.txt
echo "done" >> gpurun_out/rc_2b.txt
