# 1 GPU: forward with P released in two halves (variant 0) vs once (1): kernel tests + sustained timing.
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_api_gpu.py -q -x -p no:cacheprovider --timeout 120 > gpurun_out/fwd_pytest.log 2>&1; echo p=$?
tail -1 gpurun_out/fwd_pytest.log
for r in 1 2; do for v in 0 1 2; do
  A2D_FWD_VARIANT=$v timeout 300 python tools/kbench.py --S 131072 --only fwd --secs 6 >> gpurun_out/fwd_v$v.jsonl 2>&1
done; done
for v in 0 1 2; do A2D_FWD_VARIANT=$v timeout 300 python tools/kbench.py --S 32768 --only fwd --iters 5 >> gpurun_out/fwd_v$v.jsonl 2>&1; done
for v in 0 1 2; do echo "== v$v"; cut -c1-300 gpurun_out/fwd_v$v.jsonl; done
