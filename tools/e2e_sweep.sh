for c in 1 2 4 8 16; do
  python bench.py --skip-extras --steps 5 --e2e-chunk $c --cpu-sample 1 > gpurun_out/e2e_c$c.json 2> gpurun_out/e2e_c$c.err
done
