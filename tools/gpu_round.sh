# Round evidence on one B200: smoke, GPU tests, the default bench line, the ncu
# launch list, and one `ncu --set full` capture of a whole Schwarz iteration's
# hot kernels (summarised on the box: the report itself stays in /tmp), plus a
# small full report of the dominant kernel.  LABEL names the build; NCU_ONLY=1
# skips smoke / tests / bench.
mkdir -p gpurun_out
: > gpurun_out/rc.txt
nvidia-smi > gpurun_out/smi.txt 2>&1
if [ -z "${NCU_ONLY:-}" ]; then
  python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/rc.txt
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc.txt
  timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/rc.txt
fi
# ncu cannot profile the kernels of a graph with a conditional (WHILE) node: the
# profiled runs replay each Schwarz iteration as a plain graph (same kernels)
export YY_GRAPH=1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -s 3000 -c 2500 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc $?" >> gpurun_out/rc.txt
python tools/ncu_launches.py gpurun_out/launches.csv > gpurun_out/launches.md 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_line|k_resid|k_pres|k_interp" -s 3000 -c 40 -f -o /tmp/prof_iter $B > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc $?" >> gpurun_out/rc.txt
python tools/ncu_full_summary.py /tmp/prof_iter.ncu-rep > gpurun_out/ncu_full.md 2>&1
python tools/ncu_traffic.py /tmp/prof_iter.ncu-rep "${LABEL:-}" > gpurun_out/traffic.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_resid<.int.3, .int.2" -s 40 -c 1 -f -o gpurun_out/prof_top $B > gpurun_out/ncu3.log 2>&1
echo "ncu3 rc $?" >> gpurun_out/rc.txt
