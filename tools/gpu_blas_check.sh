timeout 900 python -m pytest tests/test_blas_gpu.py tests/test_reduction_gpu.py tests/test_fullwidth_gpu.py tests/test_robustness_gpu.py tests/test_host_gpu.py -q -x > gpurun_out/tests_blas_small.txt 2>&1
timeout 600 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so > gpurun_out/ab_light_blas7.txt 2>&1
timeout 700 python tools/stress.py 37 300 > gpurun_out/stress_r02_seed37.txt 2>&1
