"""CPU oracle for the 2D-Attention hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference functional model
(``/root/reference/pkg/src/attn2d``, numpy 2.3.5, Python 3.12) used as the
parity checker for the B200 CUDA path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it;
the product package never does (and fails loudly if its CUDA library is
missing instead of falling back here).

Parity pinned: ``tests/golden/*.npz`` hold outputs produced by importing the
reference itself (``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py``
checks this restatement against every one of them plus the reference's own
known-answer tests (zig-zag stripes, scatter layout, ring schedules).

Numerics follow the reference exactly:
* scale 1/sqrt(d); scores computed, then position mask ``k_pos <= q_pos``
  (``oracle.py:69-76``);
* stable softmax with natural-log LSE; rows with no admitted key give zero
  output and LSE = -inf, never NaN (``oracle.py:53-66``);
* GQA: query head h reads KV head h // G (``oracle.py:45-50``);
* backward: dV = P^T dO, dP = dO V^T, dS = P*(dP - rowsum(dP*P)),
  dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d), KV grads summed over the G
  sharing heads (``oracle.py:127-152``);
* merge: logaddexp of LSEs, -inf weights are 0 (``oracle.py:104-124``).
Everything is computed in float64 (the reference promotes f32 inputs to f64
after the QK^T product under numpy 2; we feed bf16-rounded
inputs as f64 so the comparison isolates kernel error).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Dense:
    """(H, T, d) values + (T,) original positions (ref ``oracle.py:15-34``)."""

    values: np.ndarray
    positions: np.ndarray


@dataclass(frozen=True)
class Block:
    """Normalised partial output + natural-log LSE (ref ``oracle.py:37-42``)."""

    out: np.ndarray
    lse: np.ndarray


def philox_qkv(seed: int, heads: int, kv_heads: int, tokens: int, head_dim: int):
    """q, k, v ~ N(0,1) drawn in that order from Philox(seed).

    Same stream as the reference fixtures (``tests/conftest.py:7-23``).
    """
    rng = np.random.Generator(np.random.Philox(seed))
    q = rng.standard_normal((heads, tokens, head_dim))
    k = rng.standard_normal((kv_heads, tokens, head_dim))
    v = rng.standard_normal((kv_heads, tokens, head_dim))
    return q, k, v


def _group(n_q: int, n_kv: int) -> int:
    if n_q % n_kv:
        raise ValueError(f"{n_q} query heads not divisible by {n_kv} kv heads")
    return n_q // n_kv


def _masked_scores(q, k, q_pos, k_pos, causal):
    """(H, Tq, Tk) scaled scores with -inf where the causal mask rejects."""
    g = _group(q.shape[0], k.shape[0])
    kk = np.repeat(k, g, axis=0)
    s = np.matmul(q, kk.transpose(0, 2, 1)) * (1.0 / math.sqrt(q.shape[-1]))
    if causal:
        keep = k_pos[None, :] <= q_pos[:, None]
        s = np.where(keep[None], s, -np.inf)
    return s


def _softmax_lse(s):
    m = s.max(axis=-1)
    m0 = np.where(np.isneginf(m), 0.0, m)
    e = np.exp(s - m0[..., None])
    e = np.where(np.isneginf(s), 0.0, e)
    z = e.sum(axis=-1)
    live = z > 0
    zs = np.where(live, z, 1.0)
    lse = np.where(live, m0 + np.log(zs), -np.inf)
    return e / zs[..., None], lse


def attention(q, k, v, q_pos, k_pos, causal=False):
    """Returns (out (H,Tq,d), lse (H,Tq)) — ref ``full_attention`` (oracle.py:79-94)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    if k.shape != v.shape:
        raise ValueError("K and V shapes differ")
    p, lse = _softmax_lse(_masked_scores(q, k, q_pos, k_pos, causal))
    vv = np.repeat(v, _group(q.shape[0], k.shape[0]), axis=0)
    return np.matmul(p, vv), lse


def attention_rows(q, k, v, q_pos, k_pos, rows, causal=False):
    """Oracle restricted to a subset of query rows (exact: the mask compares
    carried positions, ref ``test_oracle.py:79-85``). Lets S >= 32K be checked
    without the H*S^2 score tensor."""
    return attention(q[:, rows], k, v, q_pos[rows], k_pos, causal)


def attention_grads(q, k, v, d_out, q_pos, k_pos, causal=False):
    """(dq, dk, dv) — ref ``attention_backward`` (oracle.py:127-152)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    d_out = np.asarray(d_out, np.float64)
    if d_out.shape != q.shape:
        raise ValueError("d_out must match Q's shape")
    n_q, n_kv = q.shape[0], k.shape[0]
    g = _group(n_q, n_kv)
    scale = 1.0 / math.sqrt(q.shape[-1])
    p, _ = _softmax_lse(_masked_scores(q, k, q_pos, k_pos, causal))
    kk = np.repeat(k, g, axis=0)
    vv = np.repeat(v, g, axis=0)
    dv_r = np.matmul(p.transpose(0, 2, 1), d_out)
    dp = np.matmul(d_out, vv.transpose(0, 2, 1))
    ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True))
    dq = np.matmul(ds, kk) * scale
    dk_r = np.matmul(ds.transpose(0, 2, 1), q) * scale
    fold = (n_kv, g) + dk_r.shape[1:]
    return dq, dk_r.reshape(fold).sum(axis=1), dv_r.reshape(fold).sum(axis=1)


def attention_grads_rows(q, k, v, d_out_rows, q_pos, k_pos, rows, causal=False, bf16_ops=False):
    """dQ restricted to query rows ``rows`` — ref ``attention_backward``
    (oracle.py:127-152) evaluated on those rows only. Exact: every quantity of a
    dQ row (P, dP = dO V^T, row = sum(dP*P) at oracle.py:145, dS, dS K) depends
    on that row alone. ``d_out_rows`` is (H, len(rows), d)."""
    q = np.asarray(q, np.float64)[:, rows]
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    do = np.asarray(d_out_rows, np.float64)
    g = _group(q.shape[0], k.shape[0])
    scale = 1.0 / math.sqrt(q.shape[-1])
    p, _ = _softmax_lse(_masked_scores(q, k, np.asarray(q_pos)[rows], k_pos, causal))
    kk = np.repeat(k, g, axis=0)
    dp = np.matmul(do, np.repeat(v, g, axis=0).transpose(0, 2, 1))
    ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True))
    if bf16_ops:  # dS enters the dQ GEMM as bf16 in the kernel
        ds = bf16_round(ds)
    return np.matmul(ds, kk) * scale


def bf16_round(x):
    """Round to the nearest bf16 (ties to even), returned as f64: emulates the
    bf16 operands an MMA-based kernel feeds its tensor cores."""
    x32 = np.ascontiguousarray(np.asarray(x, np.float32))
    b = x32.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def attention_key_grads(q, k, v, d_out, q_pos, k_pos, keys, lse, delta, causal=False, bf16_ops=False):
    """(dK, dV) restricted to key columns ``keys`` — ref ``attention_backward``
    (oracle.py:127-152) on those columns. A key column needs every query row's
    softmax statistics: ``lse`` (H, Tq) natural log (= the oracle's LSE) and
    ``delta`` (H, Tq) = rowsum(dP*P) (oracle.py:145; equals rowsum(dO*O)). With
    those given, P[:, keys] = exp(S[:, keys] - lse) is exact, and
    dK = dS^T Q / sqrt(d), dV = P^T dO summed over the G sharing query heads
    (oracle.py:149-151)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)[:, keys]
    v = np.asarray(v, np.float64)[:, keys]
    do = np.asarray(d_out, np.float64)
    n_q, n_kv = q.shape[0], k.shape[0]
    g = _group(n_q, n_kv)
    scale = 1.0 / math.sqrt(q.shape[-1])
    s = _masked_scores(q, k, q_pos, np.asarray(k_pos)[keys], causal)
    lse = np.asarray(lse, np.float64)
    live = np.isfinite(lse)
    p = np.exp(s - np.where(live, lse, 0.0)[..., None])
    p = np.where(np.isneginf(s) | ~live[..., None], 0.0, p)
    dp = np.matmul(do, np.repeat(v, g, axis=0).transpose(0, 2, 1))
    ds = p * (dp - np.asarray(delta, np.float64)[..., None])
    if bf16_ops:  # the kernel's precision policy: P and dS enter the dV / dK GEMMs as bf16
        p, ds = bf16_round(p), bf16_round(ds)
    dk_r = np.matmul(ds.transpose(0, 2, 1), q) * scale
    dv_r = np.matmul(p.transpose(0, 2, 1), do)
    fold = (n_kv, g) + dk_r.shape[1:]
    return dk_r.reshape(fold).sum(axis=1), dv_r.reshape(fold).sum(axis=1)


def empty_block(heads, tokens, head_dim):
    return Block(np.zeros((heads, tokens, head_dim)),
                 np.full((heads, tokens), -np.inf))


def block_update(acc: Block, blk: Block) -> Block:
    """Online-softmax fold (ref ``oracle.py:111-124``)."""
    if acc.out.shape != blk.out.shape:
        raise ValueError("block shapes differ")
    new = np.logaddexp(acc.lse, blk.lse)
    ref = np.where(np.isneginf(new), 0.0, new)

    def wt(l):
        return np.where(np.isneginf(l), 0.0, np.exp(l - ref))

    out = acc.out * wt(acc.lse)[..., None] + blk.out * wt(blk.lse)[..., None]
    return Block(out, new)


# ----------------------------------------------------------------------------
# layout (ref sharding.py) — integer index maps, bit-exact
# ----------------------------------------------------------------------------

def zigzag(seq_len, d_cp):
    """(perm, inv) — ref ``zigzag_reorder`` (sharding.py:33-53)."""
    if seq_len % (2 * d_cp):
        raise ValueError(f"S={seq_len} not divisible by 2*d_cp={2 * d_cp}")
    sig = seq_len // (2 * d_cp)
    order = []
    for j in range(d_cp):
        order += [j, 2 * d_cp - 1 - j]
    perm = np.concatenate([np.arange(s * sig, (s + 1) * sig) for s in order])
    inv = np.argsort(perm)
    return perm, inv


def rank_of(hp, cp, d_hp, d_cp, head_first=True):
    """ref ``RankGrid.rank_of`` (config.py:155-158)."""
    return cp * d_hp + hp if head_first else hp * d_cp + cp


def shard(x: Dense, d_hp, d_cp, head_first=True):
    """SeqSharded chunks by global rank — ref ``shard_sequence`` (sharding.py:56-79).

    Assumes ascending positions (the reference's fast path)."""
    s = x.values.shape[1]
    if s % (2 * d_hp * d_cp):
        raise ValueError("S not divisible by 2*d_sp")
    perm, _ = zigzag(s, d_cp)
    c, l = s // d_cp, s // (d_hp * d_cp)
    out = [None] * (d_hp * d_cp)
    for j in range(d_cp):
        for i in range(d_hp):
            tok = perm[j * c + i * l: j * c + (i + 1) * l]
            idx = np.searchsorted(x.positions, tok)
            out[rank_of(i, j, d_hp, d_cp, head_first)] = Dense(
                x.values[:, idx].copy(), x.positions[idx].copy())
    return out


def replicate_kv(chunks, kv_heads, d_hp, heads):
    """ref ``kv_replicate`` (sharding.py:109-128)."""
    if d_hp > heads:
        raise ValueError(f"d_hp={d_hp} exceeds H={heads}")
    target = kv_heads if d_hp <= kv_heads else math.lcm(kv_heads, d_hp)
    rep = target // kv_heads
    if rep == 1:
        return chunks
    return [Dense(np.repeat(c.values, rep, axis=0), c.positions) for c in chunks]


def scatter(chunks, d_hp, d_cp, head_first=True):
    """SeqSharded -> HeadSharded — ref ``seq_alltoall_scatter`` (sharding.py:131-152)."""
    h = chunks[0].values.shape[0]
    if h % d_hp:
        raise ValueError(f"{h} heads not divisible by d_hp={d_hp}")
    per = h // d_hp
    out = [None] * (d_hp * d_cp)
    for j in range(d_cp):
        grp = [chunks[rank_of(i, j, d_hp, d_cp, head_first)] for i in range(d_hp)]
        vals = np.concatenate([g.values for g in grp], axis=1)
        pos = np.concatenate([g.positions for g in grp])
        for i in range(d_hp):
            out[rank_of(i, j, d_hp, d_cp, head_first)] = Dense(
                vals[i * per:(i + 1) * per].copy(), pos.copy())
    return out


def gather(chunks, d_hp, d_cp, head_first=True):
    """HeadSharded -> SeqSharded — ref ``seq_alltoall_gather`` (sharding.py:155-169)."""
    t = chunks[0].values.shape[1] // d_hp
    out = [None] * (d_hp * d_cp)
    for j in range(d_cp):
        vals = np.concatenate(
            [chunks[rank_of(i, j, d_hp, d_cp, head_first)].values
             for i in range(d_hp)], axis=0)
        pos = chunks[rank_of(0, j, d_hp, d_cp, head_first)].positions
        for i in range(d_hp):
            out[rank_of(i, j, d_hp, d_cp, head_first)] = Dense(
                vals[:, i * t:(i + 1) * t].copy(), pos[i * t:(i + 1) * t].copy())
    return out


def unshard_seq(chunks):
    """SeqSharded -> natural order — ref ``unshard`` (sharding.py:91-106)."""
    vals = np.concatenate([c.values for c in chunks], axis=1)
    pos = np.concatenate([c.positions for c in chunks])
    order = np.argsort(pos, kind="stable")
    return Dense(vals[:, order], pos[order])


def ring_sources(d_cp, w):
    """[cp_rank][step] -> source — ref ``build_ring_schedule`` (ring.py:41-61)."""
    if w < 1 or d_cp % w:
        raise ValueError(f"inner ring size {w} must divide d_cp={d_cp}")
    n = d_cp // w
    return [[((j // w - o) % n) * w + (j % w - t) % w
             for o in range(n) for t in range(w)] for j in range(d_cp)]


def double_ring(qs, ks, vs, d_cp, w, causal):
    """Per-CP-rank folded Blocks — ref ``run_double_ring`` (ring.py:64-79)."""
    res = []
    for j, q in enumerate(qs):
        acc = empty_block(*q.values.shape)
        for s in ring_sources(d_cp, w)[j]:
            o, l = attention(q.values, ks[s].values, vs[s].values,
                             q.positions, ks[s].positions, causal)
            acc = block_update(acc, Block(o, l))
        res.append(acc)
    return res


def two_d_attention(q: Dense, k: Dense, v: Dense, heads, kv_heads, d_hp, d_cp,
                    w, head_first=True, causal=False):
    """Alg. 1 pipeline — ref ``run_2d_attention`` (ring.py:82-119)."""
    qs = shard(q, d_hp, d_cp, head_first)
    ks = replicate_kv(shard(k, d_hp, d_cp, head_first), kv_heads, d_hp, heads)
    vs = replicate_kv(shard(v, d_hp, d_cp, head_first), kv_heads, d_hp, heads)
    ql, kl, vl = (scatter(x, d_hp, d_cp, head_first) for x in (qs, ks, vs))
    outs = [None] * (d_hp * d_cp)
    for i in range(d_hp):
        ranks = [rank_of(i, j, d_hp, d_cp, head_first) for j in range(d_cp)]
        blocks = double_ring([ql[r] for r in ranks], [kl[r] for r in ranks],
                             [vl[r] for r in ranks], d_cp, w, causal)
        for r, b in zip(ranks, blocks):
            outs[r] = Dense(b.out, ql[r].positions)
    return unshard_seq(gather(outs, d_hp, d_cp, head_first))
