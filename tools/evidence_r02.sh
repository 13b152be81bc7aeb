# Round-2 evidence on one B200: ncu --set full summaries of the kernels the
# bench line reports (special-form NTT passes, BLAS vmul/axpy at each width,
# the generic Barrett vmul for comparison) and the launch list of the bench.
set -x
mkdir -p gpurun_out/ncu
timeout 120 python tools/diag_stream.py > gpurun_out/r02_diag_stream.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt_ -c 2 -o gpurun_out/ncu/r02_ntt python tools/workload.py ntt --reps 1 > gpurun_out/ncu_ntt.log 2>&1
for spec in "vmul 256" "axpy 256" "vmul 128" "vmul 384" "vmul 768" "vadd 256"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none -k regex:blas_kernel -c 1 -o /tmp/r02_$1_$2 python tools/workload.py $1 --bits $2 --reps 1 > gpurun_out/ncu_$1_$2.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:blas_kernel -c 1 -o /tmp/r02_vmul_256_barrett python tools/workload.py vmul --bits 256 --reps 1 --reduction barrett > gpurun_out/ncu_vmul_256_barrett.log 2>&1
(python tools/ncu_summary.py gpurun_out/ncu/r02_ntt.ncu-rep; for f in /tmp/r02_*.ncu-rep; do echo "# $f"; python tools/ncu_summary.py $f; done) > gpurun_out/r02_ncu_summary.jsonl 2>&1
ncu -i gpurun_out/ncu/r02_ntt.ncu-rep --page raw --csv > gpurun_out/r02_ntt_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-extras --cpu-sample 1 > gpurun_out/r02_bench_under_ncu.log 2>&1
