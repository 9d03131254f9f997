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


def sampled_check(a, op, rank, qt, kt, vt, dot, out, dq, dk, dv, lse=None):
    """Gather the SeqSharded outputs (and the HeadSharded LSE of the plain
    path) to global natural order on the GPU; rank 0 checks sampled rows/keys
    of the first and last KV-head groups against the f64 oracle."""
    from oracle import sampled

    world = dist.get_world_size()

    def gather_dev(x):
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x.contiguous())
        return unshard_global(parts, op)

    O, DQ, DK, DV = (gather_dev(x) for x in (out, dq, dk, dv))
    LSE = None
    if lse is None and op.saved is not None and not a.fused_qkv and not a.native:
        lse = op.saved[3]
    if lse is not None:
        lse = lse.contiguous()  # HeadSharded (Hl, C): heads hp*Hl.., positions of CP chunk cp
        parts = [torch.empty_like(lse) for _ in range(world)]
        dist.all_gather(parts, lse)
        LSE = torch.empty((a.heads, a.seq), dtype=torch.float32, device=lse.device)
        for r, part in enumerate(parts):
            hp, cp = op.grid.coords_of(r)
            idx = op.plans[cp].pos.long()
            LSE[hp * op.Hl:(hp + 1) * op.Hl][:, idx] = part
    res = {}
    if rank == 0:
        res = sampled.check(qt, kt, vt, dot, O, DQ, DK, DV, LSE, causal=bool(a.causal), n_rows=a.rows,
                            n_keys=a.keys, seed=a.seed)
        res["violations"] = sampled.passes(res)
        res["config"] = vars(a)
        res["head_groups"] = op.ng
    return res


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
    ap.add_argument("--two-layers", action="store_true",
                    help="with --native: two layers' forwards in flight before their backwards (caller-owned "
                         "saved states, stateless context); the checked layer runs first, the other in between")
    ap.add_argument("--sampled", action="store_true",
                    help="full-size check on sampled rows/keys (oracle/sampled.py) instead of the dense oracle; "
                         "inputs drawn on the GPU (torch Philox, seeded) so S >= 16K, H = 32 fit")
    ap.add_argument("--rows", type=int, default=512)
    ap.add_argument("--keys", type=int, default=256)
    ap.add_argument("--out", default="")
    a = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    model = ModelConfig(seq_len=a.seq, heads=a.heads, kv_heads=a.kv_heads, hidden=a.heads * a.dim)
    par = ParallelConfig(d_hp=a.d_hp, d_cp=a.d_cp, inner_ring=a.w, placement=Placement(a.placement))
    op = Attn2D(model, par, ClusterConfig(), causal=bool(a.causal))

    dev = torch.device("cuda", local)
    if a.sampled:
        gen = torch.Generator(device=dev).manual_seed(a.seed)
        qt = torch.randn((a.heads, a.seq, a.dim), device=dev, generator=gen).to(torch.bfloat16)
        kt = torch.randn((a.kv_heads, a.seq, a.dim), device=dev, generator=gen).to(torch.bfloat16)
        vt = torch.randn((a.kv_heads, a.seq, a.dim), device=dev, generator=gen).to(torch.bfloat16)
        dot = torch.randn((a.heads, a.seq, a.dim), device=dev, generator=gen).to(torch.bfloat16)
    elif a.golden:
        g = np.load(a.golden)
        to = lambda b: (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
        q, k, v = (to(g[n]) for n in "qkv")
        do = np.zeros_like(q)
    else:
        q, k, v = orc.philox_qkv(a.seed, a.heads, a.kv_heads, a.seq, a.dim)
        do = np.random.Generator(np.random.Philox(a.seed + 1)).standard_normal(q.shape)
    T = lambda x: torch.from_numpy(np.asarray(x, np.float32)).to(dev).to(torch.bfloat16)  # noqa: E731
    if not a.sampled:
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
        if a.two_layers:
            out, st_a = nat.forward_with_state(*args)
            args_b = [x.flip(-1).contiguous() for x in args]  # another layer's inputs
            _, st_b = nat.forward_with_state(*args_b)
            nat.backward(shard_global(dot, op).flip(-1).contiguous(), st_b)
            dq, dk, dv = nat.backward(shard_global(dot, op), st_a)
            del st_b
        else:
            out = nat.forward(*args)
            dq, dk, dv = nat.backward(shard_global(dot, op))
        nat.sync(300.0)
        nat_transport = nat.transport
        nat_lse = nat.lse_of(st_a if a.two_layers else nat.saved).clone()
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

    if a.sampled:
        res = sampled_check(a, op, rank, qt, kt, vt, dot, out, dq, dk, dv, nat_lse if a.native else None)
        if rank == 0:
            print(json.dumps(res))
            if a.out:
                with open(a.out, "w") as f:
                    json.dump(res, f)
        dist.barrier()
        dist.destroy_process_group()
        return

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
            res["native_transport"] = nat_transport
        print(json.dumps(res))
        if a.out:
            with open(a.out, "w") as f:
                json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
