# Round evidence on one B200: GPU tests, bench line, smoke, launch list of the
# bench, ncu --set full summaries of the dominant kernels (summarised on the
# box; only the NTT report is brought back, the others are ~15 MB each).
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-extras --cpu-sample 1 > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt_ -c 2 -o /tmp/r01_ntt python tools/workload.py ntt --reps 1 > gpurun_out/ncu_ntt.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:blas_kernel -c 1 -o /tmp/r01_vmul python tools/workload.py vmul --reps 1 > gpurun_out/ncu_vmul.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:blas_kernel -c 1 -o /tmp/r01_vadd python tools/workload.py vadd --reps 1 > gpurun_out/ncu_vadd.log 2>&1
(python tools/ncu_summary.py /tmp/r01_ntt.ncu-rep; python tools/ncu_summary.py /tmp/r01_vmul.ncu-rep; python tools/ncu_summary.py /tmp/r01_vadd.ncu-rep) > gpurun_out/ncu_summary.jsonl
