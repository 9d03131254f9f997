# ncu full capture of the default backward at S=32K (one launch)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:q128 -c 1 -o gpurun_out/r3_q128do1_32k \
  python tools/kbench.py --S 32768 --only bwd --iters 1 > gpurun_out/r3_ncu.log 2>&1; echo ncu=$?
