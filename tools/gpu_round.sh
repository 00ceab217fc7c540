mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/rc.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/rc.txt
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 2500 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc $?" >> gpurun_out/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_resid|k_pres|k_interp" -s 3000 -c 14 -o gpurun_out/prof $B > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc $?" >> gpurun_out/rc.txt
