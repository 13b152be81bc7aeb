mkdir -p gpurun_out
timeout 600 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so > gpurun_out/ab_light_blas5.txt 2>&1
timeout 900 python tools/ab_r02.py paper_2501_07535_b200/libwidemod_b200.so > gpurun_out/ab_r02_head.txt 2>&1
timeout 900 python -m pytest tests/test_blas_gpu.py tests/test_reduction_gpu.py tests/test_fullwidth_gpu.py -q -x > gpurun_out/tests10.txt 2>&1
