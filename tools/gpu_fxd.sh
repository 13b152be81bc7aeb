for lib in libwidemod_b200_fxd0.so libwidemod_b200.so; do
  WM_LIB_PATH=$PWD/paper_2501_07535_b200/$lib timeout 600 python tools/ab_four_step_split.py 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_fxd.txt
done
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_configs_gpu.py -q -x > gpurun_out/tests_fxd.txt 2>&1
