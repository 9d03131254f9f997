# 1 GPU, final build with backward CTA pairs: smoke, the -m gpu suite (1-GPU cases), default bench, C2, d=64 kernel.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/l2_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/l2_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/l2_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --seq 32768 --no-e2e > gpurun_out/l2_bench_c2.log 2>&1; echo c2=$?
timeout 200 python tools/kbench.py --S 131072 --D 64 --only bwd --secs 6 > gpurun_out/l2_d64.jsonl 2>&1
tail -1 gpurun_out/l2_pytest.log; tail -1 gpurun_out/l2_smoke.log; cut -c1-300 gpurun_out/l2_d64.jsonl
