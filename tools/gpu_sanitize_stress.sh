mkdir -p gpurun_out
bash tools/sanitize.sh > gpurun_out/sanitize_r02.txt 2>&1
timeout 700 python tools/stress.py 31 420 > gpurun_out/stress_r02_seed31.txt 2>&1
