"""Selective Checkpoint++ end to end on GPUs (run under torchrun).

A two-layer toy block per rank — fused QKV projection (token-major), the 2D
attention (one shared ``Attn2D`` op), output projection, residual — is
differentiated three ways: plain autograd, SC++ ``scpp.checkpoint`` per layer,
and ``torch.utils.checkpoint`` per layer. Rank 0 reports the gradient
differences of SC++ vs plain and how many attention-forward kernels each mode
launched during the backward pass (SC++: none).

    torchrun --nproc-per-node N tests/scpp_check.py --d-hp A --d-cp B --out res.json
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_18485_b200 import _lib, scpp  # noqa: E402
from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig, Placement  # noqa: E402
from paper_2406_18485_b200.dist import Attn2D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d-hp", type=int, default=1)
    ap.add_argument("--d-cp", type=int, default=1)
    ap.add_argument("--w", type=int, default=1)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--kv-heads", type=int, default=2)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, local = int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    H, Hkv, d = a.heads, a.kv_heads, a.dim
    model = ModelConfig(seq_len=a.seq, heads=H, kv_heads=Hkv, hidden=H * d)
    par = ParallelConfig(d_hp=a.d_hp, d_cp=a.d_cp, inner_ring=a.w, placement=Placement.HEAD_FIRST)
    op = Attn2D(model, par, ClusterConfig(), causal=True)
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(7)
    hid = H * d
    Wqkv = [(torch.randn(hid, (H + 2 * Hkv) * d, device=dev, generator=g) / hid ** 0.5).bfloat16()
            for _ in range(a.layers)]
    Wo = [(torch.randn(hid, hid, device=dev, generator=g) / hid ** 0.5).bfloat16() for _ in range(a.layers)]
    g2 = torch.Generator(device=dev).manual_seed(100 + rank)
    x0 = torch.randn(op.L, hid, device=dev, generator=g2).bfloat16()
    dy = torch.randn(op.L, hid, device=dev, generator=g2).bfloat16()
    attn = scpp.Attention2D(op, layout="lhd")

    def layer(x, wqkv, wo):
        qkv = (x @ wqkv).view(op.L, H + 2 * Hkv, d)
        o = attn(qkv[:, :H], qkv[:, H:H + Hkv], qkv[:, H + Hkv:])
        return x + o.reshape(op.L, hid) @ wo

    def run(mode):
        params = [w.clone().requires_grad_(True) for w in Wqkv + Wo]
        x = x0.clone().requires_grad_(True)
        h = x
        for i in range(a.layers):
            wq, wo = params[i], params[a.layers + i]
            if mode == "plain":
                h = layer(h, wq, wo)
            elif mode == "scpp":
                h = scpp.checkpoint(layer, h, wq, wo)
            else:
                h = torch.utils.checkpoint.checkpoint(layer, h, wq, wo, use_reentrant=False)
        _lib.LOG.enabled = True
        _lib.LOG.reset()
        h.backward(dy)
        torch.cuda.synchronize()
        _lib.LOG.enabled = False
        fwd_in_bwd = _lib.LOG.by_name.get("a2d_fa_fwd_chunk", 0)
        return [x.grad] + [p.grad for p in params], fwd_in_bwd, h.detach()

    ref, n_plain, y_plain = run("plain")
    got, n_scpp, y_scpp = run("scpp")
    _, n_torch, _ = run("torch")
    diffs = []
    for r, gg in zip(ref, got):
        r, gg = r.float(), gg.float()
        diffs.append(float((gg - r).norm() / max(float(r.norm()), 1e-30)))
    res = {"rank": rank, "grad_rel_l2": max(diffs), "out_max_abs": float((y_scpp.float() - y_plain.float()).abs().max()),
           "fwd_kernels_in_bwd": {"plain": n_plain, "scpp": n_scpp, "torch_checkpoint": n_torch},
           "scpp_bytes_per_layer": scpp.scpp_bytes_per_layer(op)}
    allres = [None] * dist.get_world_size()
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps(allres))
        if a.out:
            with open(a.out, "w") as f:
                json.dump(allres, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
