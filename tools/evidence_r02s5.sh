# Round-2 (session 5) evidence on one B200: GPU tests, bench + reference arm,
# ncu --set full of the TMA-staged BLAS kernel, the
# bench's launch list.
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 ) > gpurun_out/r02s5_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s5_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02s5_bench.json 2> gpurun_out/r02s5_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s5_bench_ref.json 2> gpurun_out/r02s5_bench_ref.err
timeout 400 python tools/stress.py 43 240 > gpurun_out/r02s5_stress_seed43.txt 2>&1
# (compute-sanitizer is closed on this GPU pool: the TMA kernel's parity
#  cases -- stage reuse, ragged tail, offset views, aliasing -- are in
#  tests/test_blas_gpu.py::test_tma_staged_path and the stress run above)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:blas_tma_kernel -c 1 -o gpurun_out/r02s5_tma python tools/workload.py vmul --bits 768 --reps 1 --reduction barrett --strategy karatsuba > gpurun_out/r02s5_ncu_tma.log 2>&1
python tools/ncu_summary.py gpurun_out/r02s5_tma.ncu-rep > gpurun_out/r02s5_ncu_tma.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02s5_launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-extras --cpu-sample 1 --python-bigint 0 > gpurun_out/r02s5_bench_under_ncu.log 2>&1
echo done
