mkdir -p gpurun_out
timeout 180 python tools/diag_stream3.py > gpurun_out/diag_stream3.txt 2>&1
timeout 300 python -m pytest tests/test_robustness_gpu.py -q > gpurun_out/robust_alone.txt 2>&1
timeout 600 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_ldg.so paper_2501_07535_b200/libwidemod_b200_ept2.so > gpurun_out/ab_light_blas.txt 2>&1
timeout 600 python tools/ab_four_step_split.py > gpurun_out/ab_four_step_split.txt 2>&1
timeout 900 python tools/ab_r02.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_r2m3.so > gpurun_out/ab_r2m3.txt 2>&1
