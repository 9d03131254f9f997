"""Multi-GPU parity of the SPMD 2D-Attention runtime (run under torchrun).

Every rank builds the same seeded global q, k, v, dO (bf16-rounded), runs
``Attn2D`` forward + backward on its SeqSharded chunk, and rank 0 reassembles
the global O, dQ, dK, dV and compares them with the CPU oracle (f64).

    torchrun --nproc-per-node N tests/dist_check.py --d-hp A --d-cp B --w W \
        --placement head_first --heads 8 --kv-heads 2 --seq 1024 --dim 128 --out res.json
"""

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import attn2d_oracle as orc  # noqa: E402
from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig, Placement  # noqa: E402
from paper_2406_18485_b200.dist import Attn2D, Attn2DFunction, shard_global, unshard_global  # noqa: E402


def metrics(got, ref):
    d = np.abs(got - ref)
    return (float(d.max()), float(np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-30)),
            float(np.abs(ref).max()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d-hp", type=int, required=True)
    ap.add_argument("--d-cp", type=int, required=True)
    ap.add_argument("--w", type=int, default=1)
    ap.add_argument("--placement", default="head_first")
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--causal", type=int, default=1)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--golden", default="")
    ap.add_argument("--fused-qkv", action="store_true",
                    help="token-major (L, H+2H_kv, d) fused QKV buffer, q/k/v passed as strided views, "
                         "gradients through torch.autograd (Attn2DFunction)")
    ap.add_argument("--native", action="store_true",
                    help="run the native C++ runtime (C ABI a2d_ctx_create/a2d_fwd/a2d_bwd) instead of dist.Attn2D, "
                         "and also compare it with dist.Attn2D")
    ap.add_argument("--out", default="")
    a = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    model = ModelConfig(seq_len=a.seq, heads=a.heads, kv_heads=a.kv_heads, hidden=a.heads * a.dim)
    par = ParallelConfig(d_hp=a.d_hp, d_cp=a.d_cp, inner_ring=a.w, placement=Placement(a.placement))
    op = Attn2D(model, par, ClusterConfig(), causal=bool(a.causal))

    if a.golden:
        g = np.load(a.golden)
        to = lambda b: (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
        q, k, v = (to(g[n]) for n in "qkv")
        do = np.zeros_like(q)
    else:
        q, k, v = orc.philox_qkv(a.seed, a.heads, a.kv_heads, a.seq, a.dim)
        do = np.random.Generator(np.random.Philox(a.seed + 1)).standard_normal(q.shape)
    dev = torch.device("cuda", local)
    T = lambda x: torch.from_numpy(np.asarray(x, np.float32)).to(dev).to(torch.bfloat16)  # noqa: E731
    qt, kt, vt, dot = T(q), T(k), T(v), T(do)
    if a.fused_qkv:
        H, Hkv = a.heads, a.kv_heads
        qkv = torch.cat([shard_global(x, op).transpose(0, 1) for x in (qt, kt, vt)], dim=1).contiguous()
        qkv.requires_grad_(True)
        out_tm = Attn2DFunction.apply(qkv[:, :H], qkv[:, H:H + Hkv], qkv[:, H + Hkv:], op, "lhd")
        out_tm.backward(shard_global(dot, op).transpose(0, 1))
        out = out_tm.detach().transpose(0, 1).contiguous()
        g = qkv.grad
        dq, dk, dv = (g[:, lo:hi].transpose(0, 1).contiguous()
                      for lo, hi in ((0, H), (H, H + Hkv), (H + Hkv, H + 2 * Hkv)))
    elif a.native:
        from paper_2406_18485_b200.native import NativeAttn2D
        nat = NativeAttn2D(model, par, ClusterConfig(), causal=bool(a.causal))
        args = [shard_global(x, op) for x in (qt, kt, vt)]
        out = nat.forward(*args)
        dq, dk, dv = nat.backward(shard_global(dot, op))
        ref_out = op.forward(*args)
        ref_grads = op.backward(shard_global(dot, op))
        torch.cuda.synchronize()
        vs_py = max(float((a_.float() - b_.float()).abs().max() / max(1.0, float(b_.float().abs().max())))
                    for a_, b_ in zip((out, dq, dk, dv), (ref_out,) + tuple(ref_grads)))
        nat.close()
    else:
        out = op.forward(shard_global(qt, op), shard_global(kt, op), shard_global(vt, op))
        dq, dk, dv = op.backward(shard_global(dot, op))
    torch.cuda.synchronize()

    def gather_all(x):
        parts = [torch.empty_like(x) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, x.contiguous())
        return unshard_global(parts, op).float().cpu().numpy()

    O, DQ, DK, DV = (gather_all(x) for x in (out, dq, dk, dv))
    res = {}
    if rank == 0:
        rb = lambda x: T(x).double().cpu().numpy()  # noqa: E731
        qb, kb, vb, dob = rb(q), rb(k), rb(v), rb(do)
        pos = np.arange(a.seq)
        ro, _ = orc.attention(qb, kb, vb, pos, pos, bool(a.causal))
        res["O"] = metrics(O, ro)
        if a.golden:
            key = f"out_{a.placement}"
            res["O_golden"] = metrics(O, g[key].astype(np.float64))
        else:
            rq, rk, rv = orc.attention_grads(qb, kb, vb, dob, pos, pos, bool(a.causal))
            res["dQ"], res["dK"], res["dV"] = metrics(DQ, rq), metrics(DK, rk), metrics(DV, rv)
        res["config"] = vars(a)
        res["head_groups"] = op.ng
        if a.native:
            res["native_vs_python"] = vs_py
        print(json.dumps(res))
        if a.out:
            with open(a.out, "w") as f:
                json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
