"""Selective Checkpoint++ mechanics on CPU.

The real operator needs a GPU (tests/test_dist_gpu.py::test_selective_checkpoint_pp);
here a float64 torch stand-in with the same interface (forward_with_state /
scatter_inputs / gather_output / backward) checks the record/replay logic:
same gradients as plain autograd, and the attention forward runs once per
layer under SC++ but twice under torch.utils.checkpoint.
"""

import math

import pytest

torch = pytest.importorskip("torch")

from paper_2406_18485_b200 import scpp  # noqa: E402


class FakeOp:
    """Causal GQA attention on (H, L, d) head-major tensors, single rank."""

    def __init__(self, H, Hkv, L, d):
        self.H, self.Hkv, self.Hl, self.C, self.kd, self.d = H, Hkv, H, L, d, d
        self.forward_calls = 0

    def _attn(self, q, k, v):
        G = q.shape[0] // k.shape[0]
        k, v = k.repeat_interleave(G, 0), v.repeat_interleave(G, 0)
        s = q @ k.transpose(-1, -2) / math.sqrt(self.d)
        L = q.shape[1]
        s = s.masked_fill(torch.ones(L, L, dtype=torch.bool).triu(1), float("-inf"))
        return torch.softmax(s, -1) @ v, torch.logsumexp(s, -1)

    def forward_with_state(self, q, k, v, layout="hld"):
        self.forward_calls += 1
        out, lse = self._attn(q, k, v)
        qh, kvh = self.scatter_inputs(q, k, v, layout)
        return out.detach().clone(), (qh, kvh, out.detach().clone(), lse.detach())

    def scatter_inputs(self, q, k, v, layout="hld"):
        return q.detach().clone(), torch.stack([k.detach(), v.detach()])

    def gather_output(self, out_h, layout="hld"):
        return out_h.clone()

    def backward(self, dout, layout="hld", state=None):
        qh, kvh, _, _ = state
        with torch.enable_grad():
            q, k, v = (t.clone().requires_grad_(True) for t in (qh, kvh[0], kvh[1]))
            out, _ = self._attn(q, k, v)
            return torch.autograd.grad(out, (q, k, v), dout)


H, HKV, L, D = 4, 2, 16, 8
HID = H * D


def _setup(layers=2, seed=0):
    g = torch.Generator().manual_seed(seed)
    W = [torch.randn(HID, (H + 2 * HKV) * D, generator=g, dtype=torch.float64) / HID ** 0.5 for _ in range(layers)]
    Wo = [torch.randn(HID, HID, generator=g, dtype=torch.float64) / HID ** 0.5 for _ in range(layers)]
    x = torch.randn(L, HID, generator=g, dtype=torch.float64)
    dy = torch.randn(L, HID, generator=g, dtype=torch.float64)
    return W, Wo, x, dy


def _run(mode, op, W, Wo, x0, dy):
    attn = scpp.Attention2D(op)

    def layer(x, wq, wo):
        qkv = (x @ wq).view(L, H + 2 * HKV, D).transpose(0, 1)
        o = attn(qkv[:H], qkv[H:H + HKV], qkv[H + HKV:])
        return x + o.transpose(0, 1).reshape(L, HID) @ wo

    params = [w.clone().requires_grad_(True) for w in W + Wo]
    x = x0.clone().requires_grad_(True)
    h = x
    n = len(W)
    for i in range(n):
        if mode == "plain":
            h = layer(h, params[i], params[n + i])
        elif mode == "scpp":
            h = scpp.checkpoint(layer, h, params[i], params[n + i])
        else:
            h = torch.utils.checkpoint.checkpoint(layer, h, params[i], params[n + i], use_reentrant=False)
    fwd_before = op.forward_calls
    h.backward(dy)
    return h.detach(), [x.grad] + [p.grad for p in params], op.forward_calls - fwd_before


def test_scpp_same_gradients_no_attention_recompute():
    W, Wo, x, dy = _setup()
    y0, g0, n0 = _run("plain", FakeOp(H, HKV, L, D), W, Wo, x, dy)
    op = FakeOp(H, HKV, L, D)
    y1, g1, n1 = _run("scpp", op, W, Wo, x, dy)
    _, g2, n2 = _run("torch", FakeOp(H, HKV, L, D), W, Wo, x, dy)
    assert torch.equal(y0, y1)
    for a, b, c in zip(g0, g1, g2):
        torch.testing.assert_close(b, a, rtol=1e-12, atol=1e-12)
        torch.testing.assert_close(c, a, rtol=1e-12, atol=1e-12)
    assert n0 == 0 and n1 == 0, "SC++ must not re-run the attention forward in backward"
    assert n2 == 2, "torch.utils.checkpoint recomputes each layer's attention"
    assert op.forward_calls == 2


def test_scpp_records_released_after_backward():
    W, Wo, x, dy = _setup(layers=1)
    op = FakeOp(H, HKV, L, D)
    attn = scpp.Attention2D(op)
    seen = {}

    def layer(x, wq):
        qkv = (x @ wq).view(L, H + 2 * HKV, D).transpose(0, 1)
        o = attn(qkv[:H], qkv[H:H + HKV], qkv[H + HKV:])
        seen.setdefault("records", scpp._CTX.records)
        return o.transpose(0, 1).reshape(L, HID)

    wq = W[0].clone().requires_grad_(True)
    y = scpp.checkpoint(layer, x, wq)
    recs = seen["records"]
    assert len(recs) == 1 and recs[0][0].shape == (H, L, D) and recs[0][1].shape == (H, L)
    y.backward(torch.ones_like(y))
    assert recs == [None]  # O / LSE dropped once the backward consumed them
    assert scpp._CTX.mode is None


def test_scpp_replay_mismatch_raises():
    W, Wo, x, dy = _setup(layers=1)
    op = FakeOp(H, HKV, L, D)
    attn = scpp.Attention2D(op)
    calls = {"n": 0}

    def layer(x, wq):  # calls attention twice in the forward, once in the recompute
        calls["n"] += 1
        qkv = (x @ wq).view(L, H + 2 * HKV, D).transpose(0, 1)
        o = attn(qkv[:H], qkv[H:H + HKV], qkv[H + HKV:])
        if calls["n"] == 1:
            attn(qkv[:H], qkv[H:H + HKV], qkv[H + HKV:])
        return o.transpose(0, 1).reshape(L, HID)

    y = scpp.checkpoint(layer, x, W[0].clone().requires_grad_(True))
    with pytest.raises(RuntimeError, match="fewer attention calls"):
        y.backward(torch.ones_like(y))


def test_scpp_memory_matches_reference_model():
    """Extra bytes per layer and rank = attention output (bf16) + LSE (fp32), the
    reference's "scpp" term (ref costs.py:246-248: act_input + lse)."""
    class Op:
        Hl, C, kd = 8, 65536, 128   # H=32, d_hp=4, S=128K, d_cp=2
    S, Hh, d, d_sp = 131072, 32, 128, 8
    ref = 2 * S * (Hh * d) // d_sp + 4 * S * Hh // d_sp
    assert scpp.scpp_bytes_per_layer(Op) == ref
    assert scpp.Attention2D in scpp.WHITELIST
