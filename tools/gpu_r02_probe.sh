# 1 GPU: microbenchmarks (UMMA rates, HBM variants), same-box yardstick,
# kernel tests incl. the d=64 backward, then racecheck on the small case.
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_18485_b200/csrc tools/probes/umma_rate.cu -o /tmp/umma_rate && timeout 300 /tmp/umma_rate > gpurun_out/umma_rate.log 2>&1; echo umma=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probes/hbm_probe.cu -o /tmp/hbm_probe && timeout 300 /tmp/hbm_probe > gpurun_out/hbm_probe.log 2>&1; echo hbm=$?
timeout 300 python tools/bwd_prof.py > gpurun_out/bwd_prof.json 2>&1; echo bwdprof=$?
timeout 300 python tools/bwd_prof.py --kv-heads 8 --seq 65536 > gpurun_out/bwd_prof_gqa.json 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_api_gpu.py -q -rs -p no:cacheprovider > gpurun_out/pytest_kernels.log 2>&1; echo pytest=$?
timeout 900 python tools/yardstick.py > gpurun_out/yardstick.jsonl 2> gpurun_out/yardstick.err; echo yard=$?
timeout 600 python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py > gpurun_out/racecheck.log 2>&1; echo racecheck=$?
tail -2 gpurun_out/pytest_kernels.log
