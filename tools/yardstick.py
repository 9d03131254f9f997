"""Same-box yardstick: the library attention kernels on
this image — torch SDPA with the cuDNN backend (cuDNN 9.x) and flash_attn
2.8.3 (FA2, mma.sync) — against this repo's sm_100a kernels, causal MHA,
fwd and bwd timed separately with CUDA events, same process, same clocks.

    python tools/yardstick.py [--seqs 32768 131072] [--heads 32] [--dim 128] [--iters 5]

One JSON line per (impl, S, pass). Library code is used here only as a
yardstick; it is never on the product path. FLOPs: fwd 2*S^2*H*d (causal
half of 4*S^2*H*d), bwd 2.5x fwd.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception:
        return None


def ours(q, k, v, do, iters):
    from paper_2406_18485_b200 import kernels as K
    H, S, d = q.shape
    dev = q.device
    plan = K.ChunkPlan(torch.arange(S, dtype=torch.int32, device=dev))
    scale = 1.0 / math.sqrt(d)
    lse = torch.empty((H, S), dtype=torch.float32, device=dev)
    out = torch.empty_like(q)
    dq_acc = K.dq_acc_t(H, S, dev, d)
    dk = torch.empty((H, S, d), dtype=torch.float32, device=dev)
    dv = torch.empty_like(dk)

    def fwd():
        K.fwd_chunk(q, k, v, plan, plan, True, scale, lse, None, out)

    def bwd():
        lse2, delta = K.bwd_preprocess(out, do, lse)
        dq_acc.zero_()
        K.bwd_chunk(q, k, v, do, plan, plan, lse2, delta, dq_acc, dk, dv, False, True, scale)
        K.dqt_to_bf16(dq_acc, S)
        K.to_bf16(dk)
        K.to_bf16(dv)

    fwd()
    return timed(fwd, iters), timed(bwd, iters)


def sdpa_cudnn(q, k, v, do, iters):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    qq, kk, vv = (x.unsqueeze(0).detach().requires_grad_(True) for x in (q, k, v))
    dd = do.unsqueeze(0)
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True)

        def fwd():
            torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True)

        def bwd():
            torch.autograd.grad(o, (qq, kk, vv), dd, retain_graph=True)

        return timed(fwd, iters), timed(bwd, iters)


def flash2(q, k, v, do, iters):
    from flash_attn import flash_attn_func
    qq, kk, vv = (x.transpose(0, 1).unsqueeze(0).contiguous().requires_grad_(True) for x in (q, k, v))
    dd = do.transpose(0, 1).unsqueeze(0).contiguous()
    o = flash_attn_func(qq, kk, vv, causal=True)

    def fwd():
        flash_attn_func(qq, kk, vv, causal=True)

    def bwd():
        torch.autograd.grad(o, (qq, kk, vv), dd, retain_graph=True)

    return timed(fwd, iters), timed(bwd, iters)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, nargs="+", default=[32768, 131072])
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--impls", nargs="+", default=["ours", "cudnn", "flash_attn2"])
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    impls = {"ours": ours, "cudnn": sdpa_cudnn, "flash_attn2": flash2}
    for S in a.seqs:
        g = torch.Generator(device=dev).manual_seed(S)
        q, k, v, do = (torch.randn((a.heads, S, a.dim), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
        f_fwd = 2.0 * S * S * a.heads * a.dim
        for name in a.impls:
            try:
                t_f, t_b = impls[name](q, k, v, do, a.iters)
                rec = {"impl": name, "S": S, "H": a.heads, "d": a.dim, "causal": True,
                       "fwd_ms": t_f, "bwd_ms": t_b, "fwd_tflops": f_fwd / t_f / 1e9,
                       "bwd_tflops": 2.5 * f_fwd / t_b / 1e9, "fwd_bwd_tflops": 3.5 * f_fwd / (t_f + t_b) / 1e9,
                       "clocks_after": clocks()}
            except Exception as exc:  # a library backend may refuse a shape
                rec = {"impl": name, "S": S, "error": f"{type(exc).__name__}: {exc}"[:300]}
            print(json.dumps(rec), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
