set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider --timeout 120 > gpurun_out/r3_pytest_kernels.log 2>&1; echo p=$?
tail -1 gpurun_out/r3_pytest_kernels.log
timeout 300 python tools/kbench.py --S 32768 --only bwd --iters 5 > gpurun_out/r3_b.jsonl 2>&1
timeout 300 python tools/kbench.py --S 131072 --only bwd --secs 8 >> gpurun_out/r3_b.jsonl 2>&1
for ab in 0 3; do A2D_TRACE=1 A2D_ABLATE=$ab timeout 300 python tools/bwd_prof.py > gpurun_out/r3_trace_$ab.json 2>&1; done
cat gpurun_out/r3_b.jsonl
