# 1 GPU: backward variants (A2D_BWD_VARIANT) sustained + burst, their wait
# profiles, the forward sustained, and the HBM transpose variants.
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probes/hbm_probe.cu -o /tmp/hbm_probe && timeout 300 /tmp/hbm_probe > gpurun_out/hbm_probe2.log 2>&1
for v in 0 1 2 3 0; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 >> gpurun_out/bwdvar.jsonl 2>&1
  echo "variant $v done" >> gpurun_out/bwdvar.jsonl
done
for v in 0 2 3; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/bwd_prof.py > gpurun_out/bwd_prof_v$v.json 2>&1
done
timeout 300 python tools/kbench.py --S 131072 --only fwd --secs 8 > gpurun_out/fwd_sust.jsonl 2>&1
timeout 300 python tools/kbench.py --S 32768 --iters 5 > gpurun_out/k32k.jsonl 2>&1
