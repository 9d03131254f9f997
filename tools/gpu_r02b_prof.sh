# 1 GPU: wait profile + ncu capture of the 128-query backward.
set -x
python -m paper_2406_18485_b200.build > gpurun_out/build.log 2>&1
python -m paper_2406_18485_b200.build --profile > gpurun_out/build_prof.log 2>&1; echo bp=$?
timeout 300 python tools/bwd_prof.py > gpurun_out/r3_bwd_prof_q128.json 2>&1; echo prof=$?
timeout 300 python tools/bwd_prof.py --seq 32768 > gpurun_out/r3_bwd_prof_q128_32k.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:q128 -c 1 -o gpurun_out/r3_q128_32k \
  python tools/kbench.py --S 32768 --only bwd --iters 1 > gpurun_out/r3_ncu.log 2>&1; echo ncu=$?
cat gpurun_out/r3_bwd_prof_q128.json
