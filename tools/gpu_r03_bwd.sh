# 1 GPU: the 128-query backward — kernel parity, variant timing, wait profiles.
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/r3_pytest_kernels.log 2>&1; echo p=$?
tail -1 gpurun_out/r3_pytest_kernels.log
for v in ${VARS:-0 7}; do
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 32768 --only bwd --iters 5 >> gpurun_out/r3_bwd_v$v.jsonl 2>&1
  A2D_BWD_VARIANT=$v timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 >> gpurun_out/r3_bwd_v$v.jsonl 2>&1
  A2D_BWD_VARIANT=$v timeout 300 python tools/bwd_prof.py > gpurun_out/r3_bwd_prof_v$v.json 2>&1
done
for v in ${VARS:-0 7}; do echo "== v$v"; cat gpurun_out/r3_bwd_v$v.jsonl; python -c "
import json; d=json.load(open('gpurun_out/r3_bwd_prof_v$v.json')); print(d['bwd_tflops']); [print(k, d[k]) for k in ('mma','pds','drain','tma')]"; done
