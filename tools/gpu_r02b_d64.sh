# 1 GPU: the 128-query backward at head dim 64 — kernel tests, timing vs the round-2 64-query kernel.
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_api_gpu.py -q -x -p no:cacheprovider --timeout 120 > gpurun_out/d64_pytest.log 2>&1; echo p=$?
tail -1 gpurun_out/d64_pytest.log
for v in 0 6; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 131072 --D 64 --only bwd --secs 6 >> gpurun_out/d64_bwd_v$v.jsonl 2>&1
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 32768 --D 64 --only bwd --iters 5 >> gpurun_out/d64_bwd_v$v.jsonl 2>&1
done
cat gpurun_out/d64_bwd_v*.jsonl | cut -c1-330
