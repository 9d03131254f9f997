set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -rs -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-check --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-check --no-cpu > gpurun_out/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/pytest_gpu.log
