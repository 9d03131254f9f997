# 1 GPU iteration: kernel + full-size parity tests, sustained fwd/bwd kernel timing, bench N=1.
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_parity_scale.py tests/test_api_gpu.py -q -x -p no:cacheprovider --timeout 240 > gpurun_out/it_pytest.log 2>&1; echo p=$?
tail -2 gpurun_out/it_pytest.log
timeout 120 python tools/kbench.py --S 131072 --only fwd --secs 8 > gpurun_out/it_fwd.jsonl 2>&1
timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 > gpurun_out/it_bwd.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/it_bench.log 2>&1; echo bench=$?
cat gpurun_out/it_fwd.jsonl gpurun_out/it_bwd.jsonl; tail -1 gpurun_out/it_bench.log | cut -c1-1500
