timeout 900 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_smallall.so > gpurun_out/ab_light_blas6.txt 2>&1
