# 1 GPU, round-2b build evidence (128-query backward): smoke, the whole -m gpu suite (1-GPU cases),
# the default bench (N=1, parity check on), BASELINE config 1/2 shapes, the
# native runtime, then the ncu launch list (with DRAM bytes) of the bench
# command and one ncu --set full capture of each attention kernel.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/g1_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/g1_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --seq 32768 --no-e2e > gpurun_out/g1_bench_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --seq 4096 --heads 8 --kv-heads 8 --dim 64 --steps 20 > gpurun_out/g1_bench_c1_1gpu.log 2>&1; echo c1=$?
timeout 600 python bench.py --runtime native --no-check > gpurun_out/g1_bench_native.log 2>&1; echo native=$?
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-check --no-cpu > gpurun_out/g1_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g1_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-check --no-cpu > gpurun_out/g1_ncu_launch.log 2>&1; echo ncu1=$?
timeout 300 python tools/kbench.py --S 131072 --iters 1 > gpurun_out/g1_kb_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_bwd_q128_kernel -c 1 -o gpurun_out/g1_fa_bwd -f python tools/kbench.py --S 131072 --iters 1 > gpurun_out/g1_ncu_bwd.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd_kernel -c 1 -o gpurun_out/g1_fa_fwd -f python tools/kbench.py --S 131072 --iters 1 > gpurun_out/g1_ncu_fwd.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/g1_pytest.log
