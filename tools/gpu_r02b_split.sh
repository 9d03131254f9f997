# 1 GPU: forward NP=2 (default) vs NP=4 (variant 2); backward default vs two-part P/dS release (variant 11).
# Each variant is first run once under a short timeout (a hang costs 90 s, not the call).
set -x
A2D_FWD_VARIANT=2 timeout 90 python tools/kbench.py --S 8192 --only fwd --iters 1 > gpurun_out/sp_probe_f2.log 2>&1; f2=$?; echo f2=$f2
A2D_BWD_VARIANT=11 timeout 90 python tools/kbench.py --S 8192 --only bwd --iters 1 > gpurun_out/sp_probe_b11.log 2>&1; b11=$?; echo b11=$b11
if [ $f2 = 0 ]; then A2D_FWD_VARIANT=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k fwd > gpurun_out/sp_pytest_f2.log 2>&1; echo pf2=$?; fi
if [ $b11 = 0 ]; then A2D_BWD_VARIANT=11 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k bwd > gpurun_out/sp_pytest_b11.log 2>&1; echo pb11=$?; fi
for r in 1 2; do
  if [ $f2 = 0 ]; then for v in 0 2; do A2D_FWD_VARIANT=$v timeout 200 python tools/kbench.py --S 131072 --only fwd --secs 6 >> gpurun_out/sp_fwd_v$v.jsonl 2>&1; done; fi
  if [ $b11 = 0 ]; then for v in 0 11; do A2D_BWD_VARIANT=$v timeout 200 python tools/kbench.py --S 131072 --only bwd --secs 6 >> gpurun_out/sp_bwd_v$v.jsonl 2>&1; done; fi
done
for f in gpurun_out/sp_pytest_*.log; do echo "$f $(tail -1 $f)"; done
for f in gpurun_out/sp_fwd_v*.jsonl gpurun_out/sp_bwd_v*.jsonl; do echo "== $f"; cut -c1-330 $f; done
