# 1 GPU: 128-query backward variants — parity of each, sustained timing.
set -x
for v in ${VARS:-0}; do
  A2D_BWD_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider --timeout 120 -k bwd > gpurun_out/r3_pytest_v$v.log 2>&1; echo v=$v p=$?
  tail -1 gpurun_out/r3_pytest_v$v.log
done
for r in 1 2; do for v in ${VARS:-0}; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 >> gpurun_out/r3_bwd_v$v.jsonl 2>&1
done; done
for v in ${VARS:-0}; do A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 32768 --only bwd --iters 5 >> gpurun_out/r3_bwd_v$v.jsonl 2>&1; done
for v in ${VARS:-0}; do echo "== v$v"; cat gpurun_out/r3_bwd_v$v.jsonl | cut -c1-400; done
