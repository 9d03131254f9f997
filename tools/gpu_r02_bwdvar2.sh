# 1 GPU: correctness of the new backward variants + dqt kernel, then timing.
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/v_pytest0.log 2>&1; echo p0=$?
A2D_BWD_VARIANT=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "bwd or smoke" > gpurun_out/v_pytest4.log 2>&1; echo p4=$?
A2D_BWD_VARIANT=4 timeout 900 python -m pytest tests/test_parity_scale.py -q -x -p no:cacheprovider -s -k "1x1w1 and S131072" > gpurun_out/v_scale4.log 2>&1; echo s4=$?
for v in 0 4 5 0 4; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 >> gpurun_out/bwdvar2.jsonl 2>&1
  echo "variant $v done" >> gpurun_out/bwdvar2.jsonl
done
for v in 0 4; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 32768 --iters 5 >> gpurun_out/bwdvar2_32k.jsonl 2>&1
  A2D_BWD_VARIANT=$v timeout 300 python tools/bwd_prof.py > gpurun_out/bwd_prof2_v$v.json 2>&1
done
