# 1 GPU: forward exp split (variants 3/4/0/5 = 0, 1/8, 1/4, 3/8 of the exp pairs on the FMA pipe), sustained S=128K.
for v in 3 4 0 5; do A2D_FWD_VARIANT=$v timeout 120 python tools/kbench.py --S 131072 --only fwd --secs 6 >> gpurun_out/px_fwd_v$v.jsonl 2>&1; echo v=$v rc=$?; done
for v in 3 4 0 5; do echo "== v$v"; cut -c1-300 gpurun_out/px_fwd_v$v.jsonl; done
