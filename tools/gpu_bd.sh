timeout 1200 python tools/ab_r02.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_bd.so paper_2501_07535_b200/libwidemod_b200_bd2.so > gpurun_out/ab_bd.txt 2>&1
WM_LIB_PATH=$PWD/paper_2501_07535_b200/libwidemod_b200_bd.so timeout 900 python -m pytest tests/test_blas_gpu.py tests/test_reduction_gpu.py -q -x > gpurun_out/tests_bd.txt 2>&1
