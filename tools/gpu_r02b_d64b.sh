# 1 GPU: head dim 64 backward with dQ^T in its own TMEM region (no drain wait before dP).
timeout 90 python tools/kbench.py --S 8192 --D 64 --only bwd --iters 1 > gpurun_out/d64b_probe.log 2>&1; rc=$?; echo probe=$rc
if [ $rc = 0 ]; then
  timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_api_gpu.py -q -x -p no:cacheprovider > gpurun_out/d64b_pytest.log 2>&1; echo p=$?; tail -1 gpurun_out/d64b_pytest.log
  timeout 200 python tools/kbench.py --S 131072 --D 64 --only bwd --secs 6 >> gpurun_out/d64b_bwd.jsonl 2>&1
  timeout 200 python tools/kbench.py --S 32768 --D 64 --only bwd --iters 5 >> gpurun_out/d64b_bwd.jsonl 2>&1
fi
cut -c1-300 gpurun_out/d64b_bwd.jsonl
