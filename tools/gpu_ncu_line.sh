# ncu --set full of the first launches of each line-sweep kernel class (C3, one step)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_line}" -s ${NCU_S:-3000} -c ${NCU_C:-14} -o gpurun_out/prof_line $B > gpurun_out/ncu_line.log 2>&1; echo "ncu rc $?" > gpurun_out/rc.txt
