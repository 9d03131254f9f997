# 4 GPUs, final build (forward P in quarters): the multi-rank parity suites and the N=2 / N=4 bench lines.
set -x
timeout 2400 python -m pytest tests/test_dist_gpu.py tests/test_parity_scale.py -m gpu -q -rs -p no:cacheprovider > gpurun_out/h4_pytest.log 2>&1; echo pytest=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 > gpurun_out/h4_bench_n2.log 2>&1; echo b2=$?
timeout 900 $R --nproc-per-node 4 --master-port 29572 bench.py --gpus 4 > gpurun_out/h4_bench_n4.log 2>&1; echo b4=$?
timeout 900 $R --nproc-per-node 4 --master-port 29573 bench.py --gpus 4 --d-hp 2 --d-cp 2 --w 1 > gpurun_out/h4_bench_n4_2x2.log 2>&1; echo b4b=$?
timeout 900 $R --nproc-per-node 4 --master-port 29574 bench.py --gpus 4 --runtime native > gpurun_out/h4_bench_n4_native.log 2>&1; echo b4n=$?
tail -3 gpurun_out/h4_pytest.log
