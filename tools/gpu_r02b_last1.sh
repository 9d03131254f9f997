# 1 GPU, last check of the final build: smoke, the -m gpu suite (1-GPU cases), default bench.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/l1_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/l1_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/l1_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/l1_pytest.log; tail -1 gpurun_out/l1_smoke.log
