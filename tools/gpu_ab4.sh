mkdir -p gpurun_out
timeout 180 python tools/diag_stream4.py > gpurun_out/diag_stream4.txt 2>&1
timeout 600 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_io1.so paper_2501_07535_b200/libwidemod_b200_io2.so paper_2501_07535_b200/libwidemod_b200_nopack.so > gpurun_out/ab_light_blas3.txt 2>&1
timeout 600 python tools/e2e_probe3.py > gpurun_out/e2e_probe3.txt 2>&1
timeout 600 python tools/ab_four_step_split.py > gpurun_out/ab_four_step_split3.txt 2>&1
