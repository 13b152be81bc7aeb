# Round-2 (session 5) evidence on one B200: GPU tests, bench + reference arm,
# compute-sanitizer on the TMA-staged BLAS kernel, ncu --set full of it, the
# bench's launch list.
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 ) > gpurun_out/r02s5_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s5_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02s5_bench.json 2> gpurun_out/r02s5_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s5_bench_ref.json 2> gpurun_out/r02s5_bench_ref.err
{
for tool in memcheck racecheck synccheck initcheck; do
  for spec in "vmul 768 karatsuba" "axpy 1024 schoolbook"; do
    set -- $spec
    echo "== $tool $1 $2-bit barrett $3 (blas_tma_kernel), n=2^18"
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/workload.py $1 --bits $2 --logn 18 --reps 1 --reduction barrett --strategy $3 2>&1 | tail -2
    echo "exit=$?"
  done
done
} > gpurun_out/r02s5_sanitizer.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:blas_tma_kernel -c 1 -o gpurun_out/r02s5_tma python tools/workload.py vmul --bits 768 --reps 1 --reduction barrett --strategy karatsuba > gpurun_out/r02s5_ncu_tma.log 2>&1
python tools/ncu_summary.py gpurun_out/r02s5_tma.ncu-rep > gpurun_out/r02s5_ncu_tma.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02s5_launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-extras --cpu-sample 1 --python-bigint 0 > gpurun_out/r02s5_bench_under_ncu.log 2>&1
echo done
