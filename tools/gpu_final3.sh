# Round-2 closing run on one B200 (final build): smoke, every GPU test (incl. the C3
# step-7 golden), the C3 / C5 bench lines, the ncu launch list and one full capture.
mkdir -p gpurun_out
: > gpurun_out/rc_f3.txt
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/rc_f3.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc_f3.txt
B="timeout 900 python bench.py"
$B > gpurun_out/bench_c3.log 2>&1; echo "c3 rc $?" >> gpurun_out/rc_f3.txt
$B --workload C5 --steps 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc $?" >> gpurun_out/rc_f3.txt
$B --workload C5 --steps 5 --fixed-iters 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_k10.log 2>&1; echo "c5 k10 rc $?" >> gpurun_out/rc_f3.txt
export YY_GRAPH=1
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B1 > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 3000 -c 2500 --csv --log-file gpurun_out/launches.csv $B1 > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc $?" >> gpurun_out/rc_f3.txt
python tools/ncu_launches.py gpurun_out/launches.csv > gpurun_out/launches.md 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_line|k_resid|k_pres|k_interp" -s 3000 -c 40 -f -o /tmp/prof_iter $B1 > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc $?" >> gpurun_out/rc_f3.txt
python tools/ncu_full_summary.py /tmp/prof_iter.ncu-rep > gpurun_out/ncu_full.md 2>&1
python tools/ncu_traffic.py /tmp/prof_iter.ncu-rep r02c > gpurun_out/traffic.json 2>&1
echo "done" >> gpurun_out/rc_f3.txt
