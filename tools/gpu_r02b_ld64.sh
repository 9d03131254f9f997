# 1 GPU: backward drain with two 64-column TMEM loads (variant 12) vs four 32-column ones (0).
A2D_BWD_VARIANT=12 timeout 90 python tools/kbench.py --S 8192 --only bwd --iters 1 > gpurun_out/ld_probe.log 2>&1; rc=$?; echo probe=$rc
if [ $rc = 0 ]; then
  A2D_BWD_VARIANT=12 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k bwd > gpurun_out/ld_pytest.log 2>&1; echo p=$?; tail -1 gpurun_out/ld_pytest.log
  for r in 1 2; do for v in 0 12; do A2D_BWD_VARIANT=$v timeout 200 python tools/kbench.py --S 131072 --only bwd --secs 6 >> gpurun_out/ld_bwd_v$v.jsonl 2>&1; done; done
fi
for v in 0 12; do echo "== v$v"; cut -c120-330 gpurun_out/ld_bwd_v$v.jsonl; done
