# 4 GPUs, round-2b build evidence (128-query backward): the whole -m gpu suite (1/2/4-rank cases),
# bench N=2 / N=4 (python and native runtimes), the S=128K factorisation sweep
# (head-first; placements only renumber ranks on one node, both are in the
# suite), config-4-like GQA S=256K, and config 1 on its own 2x2 w=2 grid.
set -x
nvidia-smi --query-gpu=index,name,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider --timeout 900 > gpurun_out/g4_pytest.log 2>&1; echo pytest=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 2 --master-port 29561 bench.py --gpus 2 > gpurun_out/g4_bench_n2.log 2>&1; echo b2=$?
timeout 900 $R --nproc-per-node 4 --master-port 29562 bench.py --gpus 4 > gpurun_out/g4_bench_n4.log 2>&1; echo b4=$?
timeout 900 $R --nproc-per-node 4 --master-port 29563 bench.py --gpus 4 --runtime native > gpurun_out/g4_bench_n4_native.log 2>&1; echo b4n=$?
timeout 900 $R --nproc-per-node 4 --master-port 29564 bench.py --gpus 4 --d-hp 2 --d-cp 2 --w 2 --seq 262144 --kv-heads 8 --steps 3 > gpurun_out/g4_bench_c4like_2x2.log 2>&1; echo c4a=$?
timeout 900 $R --nproc-per-node 4 --master-port 29565 bench.py --gpus 4 --d-hp 1 --d-cp 4 --w 2 --seq 262144 --kv-heads 8 --steps 3 --no-e2e > gpurun_out/g4_bench_c4like_1x4.log 2>&1; echo c4b=$?
for pl in head_first context_first; do
  timeout 600 $R --nproc-per-node 4 --master-port 29566 bench.py --gpus 4 --d-hp 2 --d-cp 2 --w 2 --placement $pl --seq 4096 --heads 8 --kv-heads 8 --dim 64 --steps 20 > gpurun_out/g4_bench_c1_$pl.log 2>&1; echo c1=$?
done
timeout 3000 python tools/sweep.py --gpus 4 --seq 131072 --steps 3 --placements head_first --out gpurun_out/g4_sweep_S128k.jsonl > gpurun_out/g4_sweep.log 2>&1; echo sweep=$?
tail -3 gpurun_out/g4_pytest.log
