"""Selective Checkpoint++ (paper §"Selective Checkpoint++",
PAPER.md:583-594; memory model ref costs.py:231-264 "scpp").

Gradient checkpointing of a whole transformer layer normally re-runs the layer
in the backward pass — including its attention, the most expensive part.
SC++ keeps the checkpoint function but puts attention on a *whitelist*:

* forward (no-grad, inside ``checkpoint``): a whitelisted attention call runs
  normally and additionally records its HeadSharded output O and LSE
  ((2·S·D + 4·S·H)/d_sp bytes per layer — the paper's figure);
* recompute (inside the backward of ``checkpoint``): the same call does NOT
  run the ring attention again. It re-scatters the recomputed q/k/v (the
  head-parallel all-to-all, needed by the attention backward anyway),
  re-gathers the recorded O, and hands (q, k, v, O, LSE) to the 2D-attention
  backward.

Whitelisted calls are ``attention(q, k, v, op)`` and modules registered with
``whitelist`` (``Attention2D`` is registered); outside ``checkpoint`` they are
plain autograd calls (``Attn2DFunction``).
"""

from __future__ import annotations

import threading

import torch

from .dist import Attn2D, Attn2DFunction


class _Ctx(threading.local):
    def __init__(self):
        self.mode = None      # None | "record" | "replay"
        self.records = None   # list of (out_h, lse) in call order
        self.cursor = 0


_CTX = _Ctx()
WHITELIST: set[type] = set()


def whitelist(cls: type) -> type:
    """Class decorator: mark a module type as SC++ whitelisted (its forward must
    route its attention through ``attention``)."""
    WHITELIST.add(cls)
    return cls


class _Replay(torch.autograd.Function):
    """Recompute-time stand-in for Attn2DFunction: no attention forward."""

    @staticmethod
    def forward(ctx, q, k, v, op: Attn2D, rec, layout: str):
        out_h, lse = rec
        qh, kvh = op.scatter_inputs(q, k, v, layout)
        ctx.op, ctx.layout, ctx.state = op, layout, (qh, kvh, out_h, lse)
        return op.gather_output(out_h, layout)

    @staticmethod
    def backward(ctx, dout):
        dq, dk, dv = ctx.op.backward(dout, ctx.layout, ctx.state)
        ctx.state = None
        return dq, dk, dv, None, None, None


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, op: Attn2D, layout: str = "hld") -> torch.Tensor:
    """Whitelisted 2D-attention call (SeqSharded in, SeqSharded out)."""
    mode = _CTX.mode
    if mode == "record":
        out, (_, _, out_h, lse) = op.forward_with_state(q, k, v, layout)
        _CTX.records.append((out_h, lse))
        return out
    if mode == "replay":
        if _CTX.cursor >= len(_CTX.records):
            raise RuntimeError("SC++ replay: more attention calls than were recorded in the forward")
        rec = _CTX.records[_CTX.cursor]
        _CTX.records[_CTX.cursor] = None  # release O / LSE once consumed
        _CTX.cursor += 1
        return _Replay.apply(q, k, v, op, rec, layout)
    return Attn2DFunction.apply(q, k, v, op, layout)


@whitelist
class Attention2D(torch.nn.Module):
    """nn.Module face of the 2D-attention operator (whitelisted for SC++)."""

    def __init__(self, op: Attn2D, layout: str = "hld"):
        super().__init__()
        self.op, self.layout = op, layout

    def forward(self, q, k, v):
        return attention(q, k, v, self.op, self.layout)


class _Checkpoint(torch.autograd.Function):
    @staticmethod
    def forward(ctx, fn, preserve_rng, *args):
        ctx.fn, ctx.preserve_rng = fn, preserve_rng
        ctx.tensor_idx = [i for i, a in enumerate(args) if torch.is_tensor(a)]
        ctx.others = [None if torch.is_tensor(a) else a for a in args]
        ctx.save_for_backward(*[args[i] for i in ctx.tensor_idx])
        if preserve_rng:
            ctx.cpu_rng = torch.get_rng_state()
            ctx.cuda_rng = torch.cuda.get_rng_state() if torch.cuda.is_initialized() else None
        records = []
        prev = (_CTX.mode, _CTX.records, _CTX.cursor)
        _CTX.mode, _CTX.records, _CTX.cursor = "record", records, 0
        try:
            with torch.no_grad():
                out = fn(*args)
        finally:
            _CTX.mode, _CTX.records, _CTX.cursor = prev
        ctx.records = records
        return out

    @staticmethod
    def backward(ctx, *grads):
        saved = ctx.saved_tensors
        args = list(ctx.others)
        for i, t in zip(ctx.tensor_idx, saved):
            d = t.detach()
            d.requires_grad_(t.requires_grad)
            args[i] = d
        prev = (_CTX.mode, _CTX.records, _CTX.cursor)
        _CTX.mode, _CTX.records, _CTX.cursor = "replay", ctx.records, 0
        try:
            with torch.random.fork_rng(devices=[torch.cuda.current_device()] if ctx.preserve_rng
                                       and ctx.cuda_rng is not None else [], enabled=ctx.preserve_rng):
                if ctx.preserve_rng:
                    torch.set_rng_state(ctx.cpu_rng)
                    if ctx.cuda_rng is not None:
                        torch.cuda.set_rng_state(ctx.cuda_rng)
                with torch.enable_grad():
                    out = ctx.fn(*args)
            if _CTX.cursor != len(ctx.records):
                raise RuntimeError("SC++ replay: fewer attention calls than were recorded in the forward")
        finally:
            _CTX.mode, _CTX.records, _CTX.cursor = prev
        ctx.records = None
        outs = out if isinstance(out, tuple) else (out,)
        pairs = [(o, g) for o, g in zip(outs, grads) if torch.is_tensor(o) and o.requires_grad and g is not None]
        if pairs:
            torch.autograd.backward([o for o, _ in pairs], [g for _, g in pairs])
        return (None, None) + tuple(a.grad if torch.is_tensor(a) and a.requires_grad else None for a in args)


def checkpoint(fn, *args, preserve_rng_state: bool = True):
    """SC++ checkpoint of ``fn(*args)``: activations are dropped and recomputed
    in the backward, except whitelisted attention, whose O and LSE are kept and
    not recomputed. Gradients flow to tensor ``args`` and to parameters used by
    ``fn`` (reentrant semantics, like torch.utils.checkpoint(use_reentrant=True))."""
    return _Checkpoint.apply(fn, preserve_rng_state, *args)


def scpp_bytes_per_layer(op: Attn2D) -> int:
    """Extra memory SC++ keeps per layer and rank: HeadSharded O (bf16) + LSE (fp32)
    — ref costs.py:246-248 (act_input + lse)."""
    return op.Hl * op.C * op.kd * 2 + op.Hl * op.C * 4
