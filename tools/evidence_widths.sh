# ncu --set full summaries of the BLAS and NTT kernels across widths
# (summarised on the box: the reports themselves are ~15 MB each)
out=gpurun_out/ncu_summary_widths.jsonl
: > $out
for b in 128 384 768; do
  for w in vmul vadd ntt; do
    k=blas_kernel; c=1
    if [ $w = ntt ]; then k=ntt_; c=2; fi
    timeout 300 ncu --set full --clock-control none -k regex:$k -c $c -o /tmp/w_${w}$b python tools/workload.py $w --bits $b --reps 1 > /dev/null 2>&1
    python tools/ncu_summary.py /tmp/w_${w}$b.ncu-rep | sed "s/^{/{\"bits\": $b, /" >> $out
    rm -f /tmp/w_${w}$b.ncu-rep
  done
done
