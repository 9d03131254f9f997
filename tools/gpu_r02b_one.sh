# 1 GPU: backward drain with one box in flight (variant 13) vs two (0): parity, sustained timing, wait profiles.
A2D_BWD_VARIANT=13 timeout 90 python tools/kbench.py --S 8192 --only bwd --iters 1 > gpurun_out/one_probe.log 2>&1; rc=$?; echo probe=$rc
if [ $rc = 0 ]; then
  A2D_BWD_VARIANT=13 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k bwd > gpurun_out/one_pytest.log 2>&1; echo p=$?; tail -1 gpurun_out/one_pytest.log
  for r in 1 2; do for v in 0 13; do A2D_BWD_VARIANT=$v timeout 200 python tools/kbench.py --S 131072 --only bwd --secs 6 >> gpurun_out/one_bwd_v$v.jsonl 2>&1; done; done
  for v in 0 13; do A2D_BWD_VARIANT=$v timeout 200 python tools/bwd_prof.py > gpurun_out/one_prof_v$v.json 2>&1; done
fi
for v in 0 13; do echo "== v$v"; cut -c120-330 gpurun_out/one_bwd_v$v.jsonl; python -c "
import json; d=json.load(open('gpurun_out/one_prof_v$v.json')); print(round(d['bwd_tflops']), d['mma'])"; done
