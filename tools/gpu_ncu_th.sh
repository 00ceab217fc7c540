# ncu --set full of the first k_line_th launches of one C3 step (YY_GRAPH=1)
mkdir -p gpurun_out
export YY_GRAPH=1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${NCU_K:-k_line_th}" -s ${NCU_S:-200} -c ${NCU_C:-6} -f -o gpurun_out/prof_th $B > gpurun_out/ncu_th.log 2>&1; echo "ncu rc $?" > gpurun_out/rc_ncu.txt
