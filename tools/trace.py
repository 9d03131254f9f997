"""Measured Chrome trace of one 2D-attention fwd+bwd step (run under torchrun).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/trace.py --d-hp 2 --d-cp 2 --w 2 --seq 131072 --out profiles/trace.json

Writes Chrome Trace Event JSON (chrome://tracing, Perfetto): pid 0 = measured
per-rank phases (CUDA events on the compute stream), pid 1 = the planner's
prediction for the same config; prints the per-phase summary.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_18485_b200 import trace  # noqa: E402
from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig, Placement  # noqa: E402
from paper_2406_18485_b200.dist import Attn2D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d-hp", type=int, default=1)
ap.add_argument("--d-cp", type=int, default=1)
ap.add_argument("--w", type=int, default=1)
ap.add_argument("--placement", default="head_first")
ap.add_argument("--seq", type=int, default=131072)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=32)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--out", default="gpurun_out/trace.json")
a = ap.parse_args()

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
model = ModelConfig(seq_len=a.seq, heads=a.heads, kv_heads=a.kv_heads, hidden=a.heads * a.dim)
par = ParallelConfig(d_hp=a.d_hp, d_cp=a.d_cp, inner_ring=a.w, placement=Placement(a.placement))
op = Attn2D(model, par, ClusterConfig(), causal=True)
g = torch.Generator(device="cuda").manual_seed(1 + dist.get_rank())
mk = lambda h: torch.randn(h, op.L, a.dim, device="cuda", generator=g).bfloat16()  # noqa: E731
q, k, v, do = mk(a.heads), mk(a.kv_heads), mk(a.kv_heads), mk(a.heads)
for _ in range(a.warmup):
    op.forward(q, k, v)
    op.backward(do)
torch.cuda.synchronize()
dist.barrier()
op.record_times = True
op.forward(q, k, v)
op.backward(do)
torch.cuda.synchronize()
ev = op.times.events
marks = [(n, ev[0][1].elapsed_time(e)) for n, e in ev]
per_rank = [None] * dist.get_world_size()
dist.all_gather_object(per_rank, marks)
if dist.get_rank() == 0:
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    summ = trace.export(a.out, dict(enumerate(per_rank)), model, par)
    summ["config"] = vars(a)
    print(json.dumps(summ))
dist.barrier()
dist.destroy_process_group()
