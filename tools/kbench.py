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
ap.add_argument("--secs", type=float, default=0.0, help="sustained mode: repeat for this long, sample clocks")
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
dq = K.dq_acc_t(H, S, dev, D)
dk = torch.empty(Hkv, S, D, device=dev); dv = torch.empty_like(dk)
def bwd():
    K.bwd_chunk(q, k, v, do, plan, plan, lse2, delta, dq, dk, dv, False, bool(a.causal), scale)
clk = {}
def timeit(fn):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    iters = a.iters
    if a.secs > 0:  # sustained: size the run to ~secs seconds (power-capped clocks)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        iters = max(1, int(a.secs * 1000 / max(e0.elapsed_time(e1), 1e-3)))
        import subprocess, statistics, tempfile
        log = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        mon = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits", "-lms", "100"], stdout=log,
                               stderr=subprocess.DEVNULL)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    if a.secs > 0:
        mon.terminate(); mon.wait(); log.seek(0)
        rows = [l.split(",") for l in log.read().splitlines() if l.count(",") == 1]
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        pw = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        half = len(sm) // 2  # steady state: second half of the run
        clk[fn.__name__] = {"sm_mhz": statistics.median(sm[half:]) if sm else None,
                            "power_w": statistics.median(pw[half:]) if pw else None, "iters": iters}
    return e0.elapsed_time(e1) / iters
c = 0.5 if a.causal else 1.0
f_fwd = 4 * S * S * H * D * c
f_bwd = 2.5 * f_fwd
tf = timeit(fwd) if a.only != 'bwd' else 1.0
tb = timeit(bwd) if a.only != 'fwd' else 1.0
print(json.dumps({"S": S, "H": H, "Hkv": Hkv, "D": D, "causal": a.causal,
    "fwd_ms": round(tf, 3), "fwd_tflops": round(f_fwd / tf / 1e9, 1),
    "bwd_ms": round(tb, 3), "bwd_tflops": round(f_bwd / tb / 1e9, 1),
    "fwdbwd_tflops": round((f_fwd + f_bwd) / (tf + tb) / 1e9, 1), **({"clocks": clk} if clk else {})}))
