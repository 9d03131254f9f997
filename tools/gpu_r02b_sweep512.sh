# 4 GPUs: BASELINE config 5 — S=512K causal, every d_hp x d_cp factorisation at 2 and 4 GPUs (head-first;
# placements only renumber ranks on one node). Parity is covered at S<=128K by the -m gpu suite.
timeout 2400 python tools/sweep.py --gpus 2 4 --seq 524288 --steps 2 --placements head_first --bench-args=--no-check --timeout 900 --out gpurun_out/sw512_S512k.jsonl > gpurun_out/sw512.log 2>&1; echo sweep=$?
cat gpurun_out/sw512.log
