mkdir -p gpurun_out
timeout 180 python tools/diag_stream3.py > gpurun_out/diag_stream3.txt 2>&1
timeout 300 python -m pytest tests/test_robustness_gpu.py tests/test_blas_gpu.py -q -k "robust or packed or plan_creation or reference_pins or golden" > gpurun_out/robust_blas.txt 2>&1
timeout 600 python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_nopack.so > gpurun_out/ab_light_blas2.txt 2>&1
timeout 600 python tools/ab_four_step_split.py > gpurun_out/ab_four_step_split2.txt 2>&1
timeout 600 python bench.py --skip-extras > gpurun_out/bench_skip.json 2> gpurun_out/bench_skip.err
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
