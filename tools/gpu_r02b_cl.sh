# 1 GPU: backward CTA pairs with multicast Q/dO (variant 14) vs default: probe, parity, timing.
A2D_BWD_VARIANT=14 timeout 60 python tools/kbench.py --S 8192 --only bwd --iters 1 > gpurun_out/cl_probe.log 2>&1; rc=$?; echo probe=$rc
tail -3 gpurun_out/cl_probe.log
if [ $rc = 0 ]; then
  A2D_BWD_VARIANT=14 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k bwd > gpurun_out/cl_pytest.log 2>&1; echo p=$?; tail -3 gpurun_out/cl_pytest.log
  for r in 1 2; do for v in 0 14; do A2D_BWD_VARIANT=$v timeout 200 python tools/kbench.py --S 131072 --only bwd --secs 6 >> gpurun_out/cl_bwd_v$v.jsonl 2>&1; done; done
  for v in 0 14; do A2D_BWD_VARIANT=$v timeout 200 python tools/kbench.py --S 32768 --only bwd --iters 5 >> gpurun_out/cl_bwd_v$v.jsonl 2>&1; done
fi
for v in 0 14; do echo "== v$v"; cut -c100-330 gpurun_out/cl_bwd_v$v.jsonl; done
