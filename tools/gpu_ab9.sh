mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --cpu-sample 2 --extras blas four_step batched > gpurun_out/bench_2rank_dryrun.json 2> gpurun_out/bench_2rank_dryrun.err
timeout 1500 python tools/ab_r02.py paper_2501_07535_b200/libwidemod_b200.so paper_2501_07535_b200/libwidemod_b200_w2.so paper_2501_07535_b200/libwidemod_b200_kr16.so paper_2501_07535_b200/libwidemod_b200_w2kr16.so > gpurun_out/ab_wide.txt 2>&1
