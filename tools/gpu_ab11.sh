timeout 900 python tools/e2e_ab_post.py > gpurun_out/e2e_ab_ramp.txt 2>&1
