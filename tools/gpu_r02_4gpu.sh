# 4-GPU validation of the build: the whole -m gpu suite (1/2/4-rank cases run,
# 8-rank cases skip), then the bench at N=2 and N=4.
set -x
nvidia-smi --query-gpu=index,name,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider > gpurun_out/pytest_gpu_4.log 2>&1; echo pytest=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1; echo bench2=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 4 > gpurun_out/bench_n4.log 2>&1; echo bench4=$?
tail -3 gpurun_out/pytest_gpu_4.log
