# Round-2 (session 3) evidence on one B200: GPU tests, bench + reference arm,
# the bench's launch list, ncu --set full of the benched kernels.
mkdir -p gpurun_out/ncu
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/pytest_gpu_d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_d.log
timeout 900 python bench.py > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_d.json 2> gpurun_out/bench_ref_d.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02d_launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-extras --cpu-sample 1 --python-bigint 0 > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt_ -c 2 -o gpurun_out/ncu/r02d_ntt python tools/workload.py ntt --reps 1 > gpurun_out/ncu_ntt.log 2>&1
for spec in "vadd 128" "vmul 128" "vmul 256" "axpy 256" "vmul 384" "vmul 768"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none -k "regex:blas_(small_)?kernel" -c 1 -o /tmp/r02d_$1_$2 python tools/workload.py $1 --bits $2 --reps 1 > gpurun_out/ncu_$1_$2.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:scale_transpose_fx -c 1 -o /tmp/r02d_fx python tools/workload.py four_step --reps 1 > gpurun_out/ncu_fx.log 2>&1
(python tools/ncu_summary.py gpurun_out/ncu/r02d_ntt.ncu-rep; for f in /tmp/r02d_*.ncu-rep; do echo "# $f"; python tools/ncu_summary.py $f; done) > gpurun_out/r02d_ncu_summary.jsonl 2>&1
