"""Kernel-level timing of the chunk fwd/bwd kernels (CUDA events)."""
import argparse, json, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_18485_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--S", type=int, default=32768)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--Hkv", type=int, default=32)
ap.add_argument("--D", type=int, default=128)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--causal", type=int, default=1)
ap.add_argument("--only", default="")
a = ap.parse_args()
dev = torch.device("cuda")
torch.manual_seed(0)
S, H, Hkv, D = a.S, a.H, a.Hkv, a.D
q = torch.randn(H, S, D, device=dev, dtype=torch.bfloat16)
k = torch.randn(Hkv, S, D, device=dev, dtype=torch.bfloat16)
v = torch.randn(Hkv, S, D, device=dev, dtype=torch.bfloat16)
do = torch.randn(H, S, D, device=dev, dtype=torch.bfloat16)
pos = torch.arange(S, device=dev, dtype=torch.int32)
plan = K.ChunkPlan(pos)
lse = torch.empty(H, S, device=dev)
out = torch.empty(H, S, D, device=dev, dtype=torch.bfloat16)
scale = 1 / math.sqrt(D)
def fwd():
    K.fwd_chunk(q, k, v, plan, plan, bool(a.causal), scale, lse, None, out)
fwd(); torch.cuda.synchronize()
lse2, delta = K.bwd_preprocess(out, do, lse)
dq = torch.zeros(H, S, D, device=dev)
dk = torch.empty(Hkv, S, D, device=dev); dv = torch.empty_like(dk)
def bwd():
    K.bwd_chunk(q, k, v, do, plan, plan, lse2, delta, dq, dk, dv, False, bool(a.causal), scale)
def timeit(fn):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters
c = 0.5 if a.causal else 1.0
f_fwd = 4 * S * S * H * D * c
f_bwd = 2.5 * f_fwd
tf = timeit(fwd) if a.only != 'bwd' else 1.0
tb = timeit(bwd) if a.only != 'fwd' else 1.0
print(json.dumps({"S": S, "H": H, "Hkv": Hkv, "D": D, "causal": a.causal,
    "fwd_ms": round(tf, 3), "fwd_tflops": round(f_fwd / tf / 1e9, 1),
    "bwd_ms": round(tb, 3), "bwd_tflops": round(f_bwd / tb / 1e9, 1),
    "fwdbwd_tflops": round((f_fwd + f_bwd) / (tf + tb) / 1e9, 1)}))
