# 1 GPU iteration: kernel parity, sustained fwd/bwd timing, wait profiles.
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; echo p=$?
for r in 1 2; do
  timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 >> gpurun_out/it_bwd.jsonl 2>&1
  timeout 300 python tools/kbench.py --S 131072 --only fwd --secs 8 >> gpurun_out/it_fwd.jsonl 2>&1
done
timeout 300 python tools/kbench.py --S 32768 --iters 5 >> gpurun_out/it_32k.jsonl 2>&1
timeout 300 python tools/bwd_prof.py > gpurun_out/it_bwd_prof.json 2>&1
timeout 300 python tools/bwd_prof.py --pass fwd > gpurun_out/it_fwd_prof.json 2>&1
