# 4 GPUs, backward CTA pairs: the multi-rank runtime parity suite and N=2 / N=4 bench lines.
set -x
timeout 1500 python -m pytest tests/test_dist_gpu.py -m gpu -q -rs -p no:cacheprovider > gpurun_out/p4_pytest.log 2>&1; echo pytest=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29581 bench.py --gpus 2 > gpurun_out/p4_bench_n2.log 2>&1; echo b2=$?
timeout 600 $R --nproc-per-node 4 --master-port 29582 bench.py --gpus 4 > gpurun_out/p4_bench_n4.log 2>&1; echo b4=$?
timeout 600 $R --nproc-per-node 4 --master-port 29583 bench.py --gpus 4 --d-hp 2 --d-cp 2 --w 1 > gpurun_out/p4_bench_n4_2x2.log 2>&1; echo b4b=$?
tail -3 gpurun_out/p4_pytest.log
