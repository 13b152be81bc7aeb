timeout 900 python -m pytest tests/test_ntt_gpu.py tests/test_fullwidth_gpu.py tests/test_configs_gpu.py tests/test_acceptance_gpu.py -q -x > gpurun_out/tests_quick.txt 2>&1
timeout 600 python tools/ab_fullwidth_ntt.py paper_2501_07535_b200/libwidemod_b200.so >> gpurun_out/tests_quick.txt 2>&1
