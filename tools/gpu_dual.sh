timeout 900 python tools/ab_r02.py paper_2501_07535_b200/libwidemod_b200_nodual.so paper_2501_07535_b200/libwidemod_b200.so > gpurun_out/ab_dual2.txt 2>&1
timeout 900 python -m pytest tests/test_ntt_gpu.py tests/test_configs_gpu.py tests/test_acceptance_gpu.py tests/test_dist_gpu.py -q -x > gpurun_out/tests_dual2.txt 2>&1
