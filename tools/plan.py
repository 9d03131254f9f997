"""Rank (d_hp, d_cp, w, placement) for a layer with the B200-calibrated model.

    python tools/plan.py --seq 131072 --heads 32 --kv-heads 8 --gpus 8
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_18485_b200 import planner as P  # noqa: E402
from paper_2406_18485_b200.config import ModelConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=131072)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=32)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--gpus", type=int, default=8)
ap.add_argument("--top", type=int, default=10)
a = ap.parse_args()
model = ModelConfig(seq_len=a.seq, heads=a.heads, kv_heads=a.kv_heads, hidden=a.heads * a.dim)
for t, p in P.plan(model, a.gpus)[:a.top]:
    pr = P.predict(model, p)
    print(json.dumps({"d_hp": p.d_hp, "d_cp": p.d_cp, "w": p.inner_ring, "placement": p.placement.value,
                      "ms": round(t * 1e3, 2), "tflops_per_gpu": round(pr["tflops_per_gpu"], 1),
                      "a2a_ms": round(pr["t_a2a"] * 1e3, 2), "ring_exposed_ms": round(pr["t_ring_exposed"] * 1e3, 2)}))
