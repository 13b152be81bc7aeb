mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_configs_gpu.py tests/test_dist_mp_gpu.py -q > gpurun_out/tests8.txt 2>&1
timeout 600 python tools/ab_four_step_split.py > gpurun_out/ab_four_step_split4.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:scale_transpose_fx -c 1 -o /tmp/r02c_fx python tools/workload.py four_step --reps 1 > gpurun_out/ncu_fx.log 2>&1
python tools/ncu_summary.py /tmp/r02c_fx.ncu-rep > gpurun_out/r02c_fx_summary.jsonl 2>&1
