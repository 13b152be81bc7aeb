mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_robustness_gpu.py tests/test_blas_gpu.py tests/test_dist_gpu.py tests/test_configs_gpu.py -q > gpurun_out/tests5.txt 2>&1
timeout 600 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_lb8.so paper_2501_07535_b200/libwidemod_b200_lb8io1.so > gpurun_out/ab_light_blas4.txt 2>&1
timeout 300 python tools/e2e_timeline.py > gpurun_out/e2e_timeline.txt 2>&1
timeout 900 python tools/e2e_probe4.py > gpurun_out/e2e_probe4.txt 2>&1
