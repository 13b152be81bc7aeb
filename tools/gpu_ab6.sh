mkdir -p gpurun_out
timeout 900 python tools/e2e_probe4.py > gpurun_out/e2e_probe5.txt 2>&1
timeout 300 python -m pytest tests/test_host_gpu.py -q > gpurun_out/tests6.txt 2>&1
WM_HOST_POST=1 timeout 300 python -m pytest tests/test_host_gpu.py -q >> gpurun_out/tests6.txt 2>&1
