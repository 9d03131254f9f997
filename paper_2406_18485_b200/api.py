"""The reference's operator API (attn2d), executed on the B200 kernels.

Same names, argument meaning and error behaviour as
``/root/reference/pkg/src/attn2d`` (``__init__.py:4-89``) for the hot path:

    full_attention, attention_block, empty_block, block_update,
    attention_backward, zigzag_reorder, shard_sequence, unshard,
    kv_replicate, seq_alltoall_scatter, seq_alltoall_gather,
    build_ring_schedule, run_double_ring, run_2d_attention

``DenseTensor.values`` may be a numpy array or a torch tensor; compute runs on
the current CUDA device in bf16 with fp32 accumulation (the reference computes
in f64; tolerance per BASELINE.json). Layout functions are pure index shuffles
and stay bit-exact for any dtype (the SeqAlltoAll ones go through the 128-bit
permute kernel when the data is on a GPU).

This module is the *global view*: one process holds every rank's chunk and
the d_sp ranks run back to back on one GPU, exactly following the ring
schedule (useful for parity and for small problems). The SPMD runtime that
runs one rank per GPU over NCCL is ``paper_2406_18485_b200.dist``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .config import (ClusterConfig, ModelConfig, ParallelConfig, RankGrid,
                     build_rank_grid, check_config)
from .layout import zigzag_reorder
from .schedule import RingSchedule, RingStep, build_ring_schedule

__all__ = [
    "DenseTensor", "BlockResult", "ShardedSeq", "full_attention", "attention_block",
    "empty_block", "block_update", "attention_backward", "zigzag_reorder",
    "shard_sequence", "unshard", "kv_replicate", "seq_alltoall_scatter",
    "seq_alltoall_gather", "build_ring_schedule", "run_double_ring",
    "run_2d_attention", "RingSchedule", "RingStep", "SEQ_SHARDED", "HEAD_SHARDED",
]

SEQ_SHARDED = "seq"
HEAD_SHARDED = "head"


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2406_18485_b200 needs a CUDA (sm_100a) device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _as_torch(x, dtype=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t


def _positions(p) -> np.ndarray:
    if isinstance(p, torch.Tensor):
        return p.detach().cpu().numpy().astype(np.int64)
    return np.asarray(p, dtype=np.int64)


@dataclass(frozen=True)
class DenseTensor:
    """(heads, tokens, head_dim) values + original token positions (ref oracle.py:15-34)."""

    values: object
    positions: object

    def __post_init__(self):
        shape = tuple(self.values.shape)
        if len(shape) != 3:
            raise ValueError(f"expected (H, T, d) values, got {shape}")
        if tuple(np.shape(self.positions)) != (shape[1],):
            raise ValueError("positions must have one entry per token")

    @property
    def heads(self) -> int:
        return self.values.shape[0]

    @property
    def tokens(self) -> int:
        return self.values.shape[1]


@dataclass(frozen=True)
class BlockResult:
    """Normalised partial output + natural-log LSE (ref oracle.py:37-42)."""

    out: torch.Tensor  # (H, Tq, d) fp32, on device
    lse: torch.Tensor  # (H, Tq) fp32


@dataclass(frozen=True)
class ShardedSeq:
    chunks: tuple
    layout: str
    grid: RankGrid

    def chunk(self, hp_index: int, cp_index: int) -> DenseTensor:
        return self.chunks[self.grid.rank_of(hp_index, cp_index)]


# ---------------------------------------------------------------- numerics

class _Prepared:
    """Device-side, padded bf16 copy of a DenseTensor + its tile plan."""

    def __init__(self, x: DenseTensor, kd: int):
        dev = _device()
        self.d = x.values.shape[-1]
        self.t = K.pad_dim(_as_torch(x.values).to(dev, non_blocking=True), kd)
        self.plan = K.ChunkPlan(torch.as_tensor(_positions(x.positions), dtype=torch.int32, device=dev))


def _check_pair(q: DenseTensor, k: DenseTensor, v: DenseTensor):
    if tuple(k.values.shape) != tuple(v.values.shape):
        raise ValueError("K and V shapes differ")
    if not np.array_equal(_positions(k.positions), _positions(v.positions)):
        raise ValueError("K and V positions differ")
    if q.heads % k.heads != 0:
        raise ValueError(f"{q.heads} query heads not divisible by {k.heads} kv heads")
    if q.values.shape[-1] != k.values.shape[-1]:
        raise ValueError("Q and K head dims differ")


def _block(q: DenseTensor, k: DenseTensor, v: DenseTensor, causal: bool) -> BlockResult:
    _check_pair(q, k, v)
    d = q.values.shape[-1]
    kd = K.fwd_dim(d)
    qp, kp, vp = _Prepared(q, kd), _Prepared(k, kd), _Prepared(v, kd)
    H, T = q.heads, q.tokens
    lse = torch.empty((H, T), dtype=torch.float32, device=qp.t.device)
    acc = torch.empty((H, T, kd), dtype=torch.float32, device=qp.t.device)
    K.fwd_chunk(qp.t, kp.t, vp.t, qp.plan, kp.plan, causal, 1.0 / math.sqrt(d), lse, acc, None)
    return BlockResult(acc[..., :d].contiguous(), lse)


def full_attention(q: DenseTensor, k: DenseTensor, v: DenseTensor,
                   causal: bool = False) -> tuple[DenseTensor, torch.Tensor]:
    """Scaled-dot-product GQA attention with position-based causal mask
    (ref oracle.py:79-94). Returns (DenseTensor out, lse)."""
    blk = _block(q, k, v, causal)
    return DenseTensor(blk.out, np.array(_positions(q.positions))), blk.lse


def attention_block(q: DenseTensor, k: DenseTensor, v: DenseTensor,
                    causal: bool = False) -> BlockResult:
    """ref oracle.py:97-101."""
    return _block(q, k, v, causal)


def empty_block(n_heads: int, n_tokens: int, head_dim: int, dtype=None) -> BlockResult:
    """Identity of block_update: zero output, -inf lse (ref oracle.py:104-108)."""
    dev = _device()
    return BlockResult(torch.zeros((n_heads, n_tokens, head_dim), dtype=torch.float32, device=dev),
                       torch.full((n_heads, n_tokens), -math.inf, dtype=torch.float32, device=dev))


def block_update(acc: BlockResult, blk: BlockResult) -> BlockResult:
    """Online-softmax fold (ref oracle.py:111-124); returns fresh tensors."""
    if tuple(acc.out.shape) != tuple(blk.out.shape):
        raise ValueError("block shapes differ")
    dev = _device()
    out = _as_torch(acc.out).to(dev, torch.float32).clone().contiguous()
    lse = _as_torch(acc.lse).to(dev, torch.float32).clone().contiguous()
    K.merge_(out, lse, _as_torch(blk.out).to(dev, torch.float32).contiguous(),
             _as_torch(blk.lse).to(dev, torch.float32).contiguous())
    return BlockResult(out, lse)


def attention_backward(q: DenseTensor, k: DenseTensor, v: DenseTensor, d_out,
                       causal: bool = False):
    """(dQ, dK, dV) of full_attention's output (ref oracle.py:127-152)."""
    _check_pair(q, k, v)
    if tuple(d_out.shape) != tuple(q.values.shape):
        raise ValueError("d_out must match Q's shape")
    d = q.values.shape[-1]
    kd = K.fwd_dim(d)
    dev = _device()
    scale = 1.0 / math.sqrt(d)
    qp, kp, vp = _Prepared(q, kd), _Prepared(k, kd), _Prepared(v, kd)
    H, T = q.heads, q.tokens
    lse = torch.empty((H, T), dtype=torch.float32, device=dev)
    out = torch.empty((H, T, kd), dtype=torch.bfloat16, device=dev)
    K.fwd_chunk(qp.t, kp.t, vp.t, qp.plan, kp.plan, causal, scale, lse, None, out)
    do = K.pad_dim(_as_torch(d_out).to(dev), kd)
    lse2, delta = K.bwd_preprocess(out, do, lse)
    dq_acc = K.dq_acc_t(H, T, dev, kd)
    dk = torch.empty((k.heads, k.tokens, kd), dtype=torch.float32, device=dev)
    dv = torch.empty_like(dk)
    K.bwd_chunk(qp.t, kp.t, vp.t, do, qp.plan, kp.plan, lse2, delta, dq_acc, dk, dv, False, causal, scale)
    return K.dq_from_acc(dq_acc, T)[..., :d], dk[..., :d], dv[..., :d]


# ---------------------------------------------------------------- layout

def _take_tokens(values, idx: np.ndarray):
    """values[:, idx] (fresh). Device tensors with 16-byte-multiple token rows go
    through the 128-bit gather_tokens kernel (the data-loader shard of ref
    shard_sequence, sharding.py:56-79); host arrays stay numpy index shuffles."""
    if isinstance(values, torch.Tensor):
        if values.is_cuda and values.dim() >= 2 and values.shape[1] > 0 and \
                (values[0, 0].numel() * values.element_size()) % 16 == 0:
            return K.gather_tokens(values, idx)
        return values[:, torch.as_tensor(idx, device=values.device)].contiguous()
    return values[:, idx].copy()


def _cat(parts, axis):
    if isinstance(parts[0], torch.Tensor):
        return torch.cat(parts, dim=axis)
    return np.concatenate(parts, axis=axis)


def shard_sequence(x: DenseTensor, grid: RankGrid) -> ShardedSeq:
    """Global tensor -> SeqSharded chunks (ref sharding.py:56-79)."""
    s = x.tokens
    if s % (2 * grid.d_sp) != 0:
        raise ValueError(f"S={s} not divisible by 2*d_sp={2 * grid.d_sp}")
    perm, _ = zigzag_reorder(s, grid.d_cp)
    pos = _positions(x.positions)
    order = np.argsort(pos, kind="stable")
    slot_of = np.empty(int(pos.max()) + 1 if pos.size else 0, dtype=np.int64)
    slot_of[pos[order]] = order
    per, c = s // grid.d_sp, s // grid.d_cp
    chunks = [None] * grid.d_sp
    for j in range(grid.d_cp):
        for i in range(grid.d_hp):
            tok = perm[j * c + i * per: j * c + (i + 1) * per]
            idx = slot_of[tok]
            chunks[grid.rank_of(i, j)] = DenseTensor(_take_tokens(x.values, idx), pos[idx].copy())
    return ShardedSeq(tuple(chunks), SEQ_SHARDED, grid)


def unshard(sharded: ShardedSeq) -> DenseTensor:
    """Reassemble in ascending position order (ref sharding.py:91-106)."""
    grid = sharded.grid
    if sharded.layout == SEQ_SHARDED:
        vals = _cat([c.values for c in sharded.chunks], 1)
        pos = np.concatenate([_positions(c.positions) for c in sharded.chunks])
    else:
        vals = _cat([_cat([sharded.chunk(i, j).values for i in range(grid.d_hp)], 0)
                     for j in range(grid.d_cp)], 1)
        pos = np.concatenate([_positions(sharded.chunk(0, j).positions) for j in range(grid.d_cp)])
    order = np.argsort(pos, kind="stable")
    return DenseTensor(_take_tokens(vals, order), pos[order])


def kv_replicate(kv: ShardedSeq, kv_heads: int, d_hp: int, n_heads: int) -> ShardedSeq:
    """GQA head replication (ref sharding.py:109-128)."""
    if d_hp > n_heads:
        raise ValueError(f"d_hp={d_hp} exceeds H={n_heads}")
    if kv.layout != SEQ_SHARDED:
        raise ValueError("kv_replicate expects SeqSharded layout")
    target = kv_heads if d_hp <= kv_heads else math.lcm(kv_heads, d_hp)
    rep = target // kv_heads
    if rep == 1:
        return kv
    out = []
    for c in kv.chunks:
        if isinstance(c.values, torch.Tensor):
            vals = torch.repeat_interleave(c.values, rep, dim=0)
        else:
            vals = np.repeat(c.values, rep, axis=0)
        out.append(DenseTensor(vals, c.positions))
    return ShardedSeq(tuple(out), SEQ_SHARDED, kv.grid)


def _alltoall_move(group_vals, d_hp: int, to_head: bool):
    """Data movement of one HP group's SeqAlltoAll, via the permute kernel on GPU."""
    if to_head:
        # rank i' contributes [H][L][d]; rank i receives heads slice i of every peer
        n_heads = group_vals[0].shape[0]
        per = n_heads // d_hp
        out = []
        for i in range(d_hp):
            parts = [gv[i * per:(i + 1) * per] for gv in group_vals]  # peer order = token order
            out.append(_cat(parts, 1))
        return out
    # HeadSharded [Hl][C][d] per rank -> SeqSharded [H][L][d]
    c = group_vals[0].shape[1]
    t = c // d_hp
    full = _cat(list(group_vals), 0)  # [H][C][d]
    return [full[:, i * t:(i + 1) * t] for i in range(d_hp)]


def _is_gpu(v) -> bool:
    """Device tensor whose per-(peer, head) blocks the 128-bit permute kernel can move."""
    if not (isinstance(v, torch.Tensor) and v.is_cuda):
        return False
    return (v.shape[1] * v.shape[2] * v.element_size()) % 16 == 0


def seq_alltoall_scatter(x: ShardedSeq, grid: RankGrid) -> ShardedSeq:
    """SeqSharded -> HeadSharded (ref sharding.py:131-152)."""
    if x.layout != SEQ_SHARDED:
        raise ValueError("scatter expects SeqSharded layout")
    n_heads = x.chunks[0].heads
    if n_heads % grid.d_hp != 0:
        raise ValueError(f"{n_heads} heads not divisible by d_hp={grid.d_hp}")
    per = n_heads // grid.d_hp
    chunks = [None] * grid.d_sp
    for j in range(grid.d_cp):
        group = [x.chunk(i, j) for i in range(grid.d_hp)]
        pos = np.concatenate([_positions(g.positions) for g in group])
        if _is_gpu(group[0].values):
            # [peer][H][L][d] -> per destination i: [peer][per][L][d] -> [per][peer][L][d]
            for i in range(grid.d_hp):
                recv = torch.stack([g.values[i * per:(i + 1) * per] for g in group])  # the all-to-all
                out = K.permute_blocks(recv, grid.d_hp, per)
                L = group[0].tokens
                chunks[grid.rank_of(i, j)] = DenseTensor(out.view(per, grid.d_hp * L, -1), pos.copy())
        else:
            vals = _alltoall_move([g.values for g in group], grid.d_hp, True)
            for i in range(grid.d_hp):
                chunks[grid.rank_of(i, j)] = DenseTensor(vals[i], pos.copy())
    return ShardedSeq(tuple(chunks), HEAD_SHARDED, grid)


def seq_alltoall_gather(o: ShardedSeq, grid: RankGrid) -> ShardedSeq:
    """HeadSharded -> SeqSharded; exact inverse of the scatter (ref sharding.py:155-169)."""
    if o.layout != HEAD_SHARDED:
        raise ValueError("gather expects HeadSharded layout")
    chunks = [None] * grid.d_sp
    for j in range(grid.d_cp):
        group = [o.chunk(i, j) for i in range(grid.d_hp)]
        pos = _positions(group[0].positions)
        C = group[0].tokens
        L = C // grid.d_hp
        if _is_gpu(group[0].values):
            per = group[0].heads
            # pack: [per][peer][L][d] -> [peer][per][L][d] on every rank, then exchange
            packed = [K.permute_blocks(g.values.contiguous(), per, grid.d_hp).view(grid.d_hp, per, L, -1)
                      for g in group]
            for i in range(grid.d_hp):
                vals = torch.cat([packed[src][i] for src in range(grid.d_hp)], dim=0)  # the all-to-all
                chunks[grid.rank_of(i, j)] = DenseTensor(vals, pos[i * L:(i + 1) * L].copy())
        else:
            vals = _alltoall_move([g.values for g in group], grid.d_hp, False)
            for i in range(grid.d_hp):
                chunks[grid.rank_of(i, j)] = DenseTensor(vals[i], pos[i * L:(i + 1) * L].copy())
    return ShardedSeq(tuple(chunks), SEQ_SHARDED, grid)


# ---------------------------------------------------------------- ring

def run_double_ring(q_chunks, k_chunks, v_chunks, schedule: RingSchedule,
                    causal: bool = False) -> list[BlockResult]:
    """Fold every KV chunk into each CP rank's accumulator in schedule order
    (ref ring.py:64-79). The fold is the fused merge epilogue of the forward
    kernel (one launch per ring step)."""
    if not (len(q_chunks) == len(k_chunks) == len(v_chunks) == schedule.d_cp):
        raise ValueError("chunk count does not match schedule")
    d = q_chunks[0].values.shape[-1]
    kd = K.fwd_dim(d)
    scale = 1.0 / math.sqrt(d)
    ks = [_Prepared(c, kd) for c in k_chunks]
    vs = [_Prepared(c, kd) for c in v_chunks]
    results = []
    for j, q in enumerate(q_chunks):
        for c in (k_chunks[0], v_chunks[0]):
            _check_pair(q, c, c)
        qp = _Prepared(q, kd)
        H, T = q.heads, q.tokens
        lse = torch.full((H, T), -math.inf, dtype=torch.float32, device=qp.t.device)
        acc = torch.zeros((H, T, kd), dtype=torch.float32, device=qp.t.device)
        for n, step in enumerate(schedule.steps[j]):
            s = step.source
            K.fwd_chunk(qp.t, ks[s].t, vs[s].t, qp.plan, ks[s].plan, causal, scale, lse, acc, None,
                        merge=n > 0)
        results.append(BlockResult(acc[..., :d].contiguous(), lse))
    return results


def run_2d_attention(q: DenseTensor, k: DenseTensor, v: DenseTensor, model: ModelConfig,
                     par: ParallelConfig, cluster: ClusterConfig,
                     causal: bool = False) -> DenseTensor:
    """Alg. 1 (ref ring.py:82-119): validate, shard, replicate, scatter,
    double ring per HP group, gather, unshard. Global view on one GPU."""
    check_config(model, par, cluster)
    grid = build_rank_grid(par, cluster)
    dev = _device()
    to_dev = lambda x: DenseTensor(_as_torch(x.values).to(dev).to(torch.bfloat16), x.positions)  # noqa: E731
    q_sh = shard_sequence(to_dev(q), grid)
    k_sh = kv_replicate(shard_sequence(to_dev(k), grid), model.kv_heads, par.d_hp, model.heads)
    v_sh = kv_replicate(shard_sequence(to_dev(v), grid), model.kv_heads, par.d_hp, model.heads)
    ql, kl, vl = (seq_alltoall_scatter(x, grid) for x in (q_sh, k_sh, v_sh))
    schedule = build_ring_schedule(par.d_cp, par.inner_ring)
    outs = [None] * grid.d_sp
    for i in range(par.d_hp):
        res = run_double_ring([ql.chunk(i, j) for j in range(par.d_cp)],
                              [kl.chunk(i, j) for j in range(par.d_cp)],
                              [vl.chunk(i, j) for j in range(par.d_cp)], schedule, causal)
        for j, r in enumerate(res):
            outs[grid.rank_of(i, j)] = DenseTensor(r.out, ql.chunk(i, j).positions)
    gathered = seq_alltoall_gather(ShardedSeq(tuple(outs), HEAD_SHARDED, grid), grid)
    return unshard(gathered)
