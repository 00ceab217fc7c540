# ncu --set full of the dominant sweep / residual kernels of one C3 Schwarz
# iteration (report kept under gpurun_out/ for local `ncu -i` analysis), then the
# chi study (RD-E4): C3 / C5 Schwarz counts and the C2 200-step drift.
mkdir -p gpurun_out
: > gpurun_out/rc.txt
export YY_GRAPH=1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_line<.int.2, .int.1, .int.2|k_line<.int.1, .int.0, .int.2|k_line<.int.3, .int.2, .int.2|k_line<.int.3, .int.1, .int.0|k_resid<.int.3, .int.2" \
  -s 2000 -c 5 -f -o gpurun_out/${LABEL:-r02}_sweeps $B > gpurun_out/ncu.log 2>&1
echo "ncu rc $?" >> gpurun_out/rc.txt
unset YY_GRAPH
timeout 600 python tools/chi_k.py C3 5 1,10,16 > gpurun_out/chi_c3.log 2>&1; echo "chi c3 rc $?" >> gpurun_out/rc.txt
timeout 600 python tools/chi_k.py C5 3 1,16 > gpurun_out/chi_c5.log 2>&1; echo "chi c5 rc $?" >> gpurun_out/rc.txt
timeout 900 python tools/c2_drift.py 200 16 5 gpurun_out/c2_drift_chi16.json > gpurun_out/c2_chi16.log 2>&1; echo "c2 chi16 rc $?" >> gpurun_out/rc.txt
timeout 900 python tools/c2_drift.py 1000 16 50 gpurun_out/c2_drift_chi16_1000.json > gpurun_out/c2_chi16_1000.log 2>&1; echo "c2 chi16 1000 rc $?" >> gpurun_out/rc.txt
