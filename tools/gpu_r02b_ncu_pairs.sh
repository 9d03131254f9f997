# ncu --set full of the paired backward at the bench shape (one launch)
timeout 240 ncu --set full --clock-control none --import-source on -k regex:fa_bwd_q128_kernel -c 1 -o gpurun_out/pq_fa_bwd -f python tools/kbench.py --S 131072 --only bwd --iters 1 > gpurun_out/pq_ncu.log 2>&1; echo ncu=$?
