"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``attn2d`` from ``$ATTN2D_REF`` (default /root/reference/pkg/src),
feeds it seeded inputs and stores inputs + outputs as small .npz files next to
this script.  The GPU box never reads /root/reference; tests there read only
these fixtures.  bf16 payloads are stored as raw uint16 bit patterns.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("ATTN2D_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import attn2d  # noqa: E402
from attn2d import (ClusterConfig, DenseTensor, ModelConfig,  # noqa: E402
                    ParallelConfig, Placement, attention_backward,
                    block_update, build_rank_grid, build_ring_schedule,
                    full_attention, run_2d_attention, seq_alltoall_scatter,
                    shard_sequence, zigzag_reorder)
from attn2d.oracle import attention_block, empty_block  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def qkv(seed, h, hkv, t, d):
    rng = philox(seed)
    return (rng.standard_normal((h, t, d)), rng.standard_normal((hkv, t, d)),
            rng.standard_normal((hkv, t, d)))


def bf16_round(x):
    """Round-to-nearest-even to bf16; returns (float64 values, uint16 bits)."""
    f = np.asarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    bits = u.astype(np.uint16)
    back = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return back, bits


def dense(a, pos=None):
    return DenseTensor(a, np.arange(a.shape[1]) if pos is None else pos)


def small_attention():
    rec = {}
    for causal in (0, 1):
        q, k, v = qkv(42, 4, 2, 16, 8)
        out, lse = full_attention(dense(q), dense(k), dense(v), bool(causal))
        rec[f"c{causal}_q"], rec[f"c{causal}_k"], rec[f"c{causal}_v"] = q, k, v
        rec[f"c{causal}_out"], rec[f"c{causal}_lse"] = out.values, lse
    # permuted query positions (mask must follow carried positions)
    q, k, v = qkv(11, 2, 2, 10, 4)
    perm = philox(5).permutation(10)
    out, lse = full_attention(DenseTensor(q[:, perm], perm), dense(k), dense(v), True)
    rec.update(perm_q=q[:, perm], perm_pos=perm, perm_k=k, perm_v=v,
               perm_out=out.values, perm_lse=lse)
    np.savez_compressed(os.path.join(OUT, "attention_small.npz"), **rec)


def small_backward():
    rec = {}
    for seed in range(3):
        for causal in (0, 1):
            q, k, v = qkv(seed, 2, 1, 6, 4)
            dout = philox(seed + 100).standard_normal(q.shape)
            dq, dk, dv = attention_backward(dense(q), dense(k), dense(v), dout,
                                            bool(causal))
            key = f"s{seed}c{causal}"
            rec.update({f"{key}_q": q, f"{key}_k": k, f"{key}_v": v,
                        f"{key}_do": dout, f"{key}_dq": dq, f"{key}_dk": dk,
                        f"{key}_dv": dv})
    q, k, v = qkv(7, 4, 2, 64, 16)
    dout = philox(8).standard_normal(q.shape)
    dq, dk, dv = attention_backward(dense(q), dense(k), dense(v), dout, True)
    rec.update(big_q=q, big_k=k, big_v=v, big_do=dout, big_dq=dq, big_dk=dk,
               big_dv=dv)
    np.savez_compressed(os.path.join(OUT, "backward_small.npz"), **rec)


def merge_cases():
    q, k, v = qkv(9, 4, 2, 16, 8)
    rec = {"q": q, "k": k, "v": v}
    for causal in (0, 1):
        acc = empty_block(4, 16, 8)
        for b in range(4):
            sl = slice(b * 4, (b + 1) * 4)
            blk = attention_block(dense(q), DenseTensor(k[:, sl], np.arange(16)[sl]),
                                  DenseTensor(v[:, sl], np.arange(16)[sl]), bool(causal))
            rec[f"c{causal}_b{b}_out"], rec[f"c{causal}_b{b}_lse"] = blk.out, blk.lse
            acc = block_update(acc, blk)
        rec[f"c{causal}_acc_out"], rec[f"c{causal}_acc_lse"] = acc.out, acc.lse
    np.savez_compressed(os.path.join(OUT, "merge.npz"), **rec)


def layouts():
    rec = {}
    for s, d_cp in ((8, 1), (8, 2), (48, 4), (64, 8), (4096, 2), (128, 4)):
        perm, inv = zigzag_reorder(s, d_cp)
        rec[f"zz_{s}_{d_cp}_perm"], rec[f"zz_{s}_{d_cp}_inv"] = perm, inv
    x_vals = np.arange(8 * 64 * 2, dtype=np.float64).reshape(8, 64, 2)
    for d_hp, d_cp in ((1, 1), (2, 2), (4, 2), (2, 4), (1, 8), (8, 1)):
        for pl in Placement:
            grid = build_rank_grid(ParallelConfig(d_hp=d_hp, d_cp=d_cp, placement=pl),
                                   ClusterConfig())
            sh = shard_sequence(dense(x_vals), grid)
            sc = seq_alltoall_scatter(sh, grid)
            tag = f"{d_hp}x{d_cp}_{pl.value}"
            rec[f"seqpos_{tag}"] = np.stack([c.positions for c in sh.chunks])
            rec[f"headpos_{tag}"] = np.stack([c.positions for c in sc.chunks])
            rec[f"headvals_{tag}"] = np.stack([c.values for c in sc.chunks])
    for d_cp in (1, 2, 4, 8):
        for w in (x for x in range(1, d_cp + 1) if d_cp % x == 0):
            sched = build_ring_schedule(d_cp, w)
            rec[f"sched_{d_cp}_{w}"] = np.array(
                [[st.source for st in row] for row in sched.steps])
    np.savez_compressed(os.path.join(OUT, "layouts.npz"), **rec)


def pipeline_small():
    rec = {}
    q, k, v = qkv(17, 8, 2, 32, 4)
    rec.update(q=q, k=k, v=v)
    model = ModelConfig(seq_len=32, heads=8, kv_heads=2, hidden=32)
    for d_hp, d_cp, w in [(1, 1, 1), (2, 2, 2), (4, 2, 1), (8, 2, 2), (1, 8, 4), (2, 4, 4)]:
        for causal in (0, 1):
            par = ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=w)
            out = run_2d_attention(dense(q), dense(k), dense(v), model, par,
                                   ClusterConfig(), bool(causal))
            rec[f"out_{d_hp}_{d_cp}_{w}_c{causal}"] = out.values
    np.savez_compressed(os.path.join(OUT, "pipeline_small.npz"), **rec)


def gpu_cases():
    """bf16-rounded inputs at kernel-tile sizes; reference outputs as float32."""
    cases = {
        # name: (seed, H, Hkv, S, d, causal)
        "mha_d128_s256_c": (101, 2, 2, 256, 128, True),
        "gqa_d128_s384_c": (102, 4, 2, 384, 128, True),
        "mha_d64_s256_n": (103, 2, 2, 256, 64, False),
        "gqa_d128_s200_n": (104, 2, 1, 200, 128, False),
    }
    for name, (seed, h, hkv, s, d, causal) in cases.items():
        q, k, v = qkv(seed, h, hkv, s, d)
        (q, qb), (k, kb), (v, vb) = bf16_round(q), bf16_round(k), bf16_round(v)
        dout, dob = bf16_round(philox(seed + 1).standard_normal(q.shape))
        out, lse = full_attention(dense(q), dense(k), dense(v), causal)
        dq, dk, dv = attention_backward(dense(q), dense(k), dense(v), dout, causal)
        np.savez_compressed(
            os.path.join(OUT, f"gpu_{name}.npz"), q=qb, k=kb, v=vb, do=dob,
            causal=np.array(causal), out=out.values.astype(np.float32),
            lse=lse.astype(np.float32), dq=dq.astype(np.float32),
            dk=dk.astype(np.float32), dv=dv.astype(np.float32))
    # 2D pipeline at a config-1 shape (scaled down): H=8 d=64 S=512, 2x2 w=2
    q, k, v = qkv(42, 8, 8, 512, 64)
    (q, qb), (k, kb), (v, vb) = bf16_round(q), bf16_round(k), bf16_round(v)
    model = ModelConfig(seq_len=512, heads=8, kv_heads=8, hidden=512)
    rec = dict(q=qb, k=kb, v=vb)
    for pl in Placement:
        par = ParallelConfig(d_hp=2, d_cp=2, inner_ring=2, placement=pl)
        out = run_2d_attention(dense(q), dense(k), dense(v), model, par,
                               ClusterConfig(), True)
        rec[f"out_{pl.value}"] = out.values.astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "gpu_pipeline_c1s.npz"), **rec)


if __name__ == "__main__":
    print("reference attn2d from", attn2d.__file__)
    small_attention()
    small_backward()
    merge_cases()
    layouts()
    pipeline_small()
    gpu_cases()
    print("wrote fixtures to", OUT)
