# compute-sanitizer passes over small NTT / BLAS / host-pipeline / four-step workloads
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/workload.py ntt --logn 12 --batch 2 --reps 1 2>&1 | tail -3
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/workload.py ntt --logn 18 --batch 1 --reps 1 2>&1 | tail -3
done
echo "== memcheck blas"
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/workload.py vmul --logn 14 --reps 1 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/workload.py vmul --bits 384 --logn 14 --reps 1 2>&1 | tail -3
echo "== memcheck/racecheck round-2 paths (packed small-element BLAS, four-step twiddle/transpose tile)"
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/workload.py vadd --bits 128 --logn 14 --reps 1 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/workload.py four_step --logn 14 --reps 1 2>&1 | tail -3
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/workload.py four_step --logn 14 --reps 1 2>&1 | tail -3
