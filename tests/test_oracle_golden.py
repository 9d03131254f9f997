"""Pin the CPU oracle restatement to the reference's own outputs (golden .npz)
and known-answer tests. CPU only."""

import math

import numpy as np
import pytest

from conftest import bf16_bits_to_f64, golden
from oracle import attn2d_oracle as orc


def test_attention_matches_reference_small():
    g = golden("attention_small.npz")
    pos = np.arange(16)
    for c in (0, 1):
        out, lse = orc.attention(g[f"c{c}_q"], g[f"c{c}_k"], g[f"c{c}_v"], pos, pos, bool(c))
        assert np.max(np.abs(out - g[f"c{c}_out"])) <= 1e-12
        assert np.max(np.abs(np.nan_to_num(lse - g[f"c{c}_lse"]))) <= 1e-12
        assert np.array_equal(np.isneginf(lse), np.isneginf(g[f"c{c}_lse"]))
    out, lse = orc.attention(g["perm_q"], g["perm_k"], g["perm_v"], g["perm_pos"],
                             np.arange(10), True)
    assert np.max(np.abs(out - g["perm_out"])) <= 1e-12


def test_backward_matches_reference_small():
    g = golden("backward_small.npz")
    for seed in range(3):
        for c in (0, 1):
            key = f"s{seed}c{c}"
            pos = np.arange(6)
            dq, dk, dv = orc.attention_grads(g[f"{key}_q"], g[f"{key}_k"], g[f"{key}_v"],
                                             g[f"{key}_do"], pos, pos, bool(c))
            for a, b in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
                assert np.max(np.abs(a - g[f"{key}_{b}"])) <= 1e-12
    pos = np.arange(64)
    dq, dk, dv = orc.attention_grads(g["big_q"], g["big_k"], g["big_v"], g["big_do"],
                                     pos, pos, True)
    for a, b in ((dq, "big_dq"), (dk, "big_dk"), (dv, "big_dv")):
        assert np.max(np.abs(a - g[b])) <= 1e-10


def test_merge_matches_reference():
    g = golden("merge.npz")
    pos = np.arange(16)
    for c in (0, 1):
        acc = orc.empty_block(4, 16, 8)
        for b in range(4):
            sl = slice(b * 4, (b + 1) * 4)
            o, l = orc.attention(g["q"], g["k"][:, sl], g["v"][:, sl], pos, pos[sl], bool(c))
            assert np.max(np.abs(o - g[f"c{c}_b{b}_out"])) <= 1e-12
            acc = orc.block_update(acc, orc.Block(o, l))
        assert np.max(np.abs(acc.out - g[f"c{c}_acc_out"])) <= 1e-12
        assert np.max(np.abs(acc.lse - g[f"c{c}_acc_lse"])) <= 1e-12


def test_self_merge_adds_ln2():
    q, k, v = orc.philox_qkv(2, 2, 1, 4, 4)
    pos = np.arange(4)
    o, l = orc.attention(q, k, v, pos, pos)
    m = orc.block_update(orc.Block(o, l), orc.Block(o, l))
    assert np.allclose(m.out, o) and np.allclose(m.lse, l + math.log(2))


def test_layouts_match_reference():
    g = golden("layouts.npz")
    for s, d_cp in ((8, 1), (8, 2), (48, 4), (64, 8), (4096, 2), (128, 4)):
        perm, inv = orc.zigzag(s, d_cp)
        assert np.array_equal(perm, g[f"zz_{s}_{d_cp}_perm"])
        assert np.array_equal(inv, g[f"zz_{s}_{d_cp}_inv"])
    x = orc.Dense(np.arange(8 * 64 * 2, dtype=np.float64).reshape(8, 64, 2), np.arange(64))
    for d_hp, d_cp in ((1, 1), (2, 2), (4, 2), (2, 4), (1, 8), (8, 1)):
        for hf, name in ((True, "head_first"), (False, "context_first")):
            tag = f"{d_hp}x{d_cp}_{name}"
            sh = orc.shard(x, d_hp, d_cp, hf)
            sc = orc.scatter(sh, d_hp, d_cp, hf)
            assert np.array_equal(np.stack([c.positions for c in sh]), g[f"seqpos_{tag}"])
            assert np.array_equal(np.stack([c.positions for c in sc]), g[f"headpos_{tag}"])
            assert np.array_equal(np.stack([c.values for c in sc]), g[f"headvals_{tag}"])
            back = orc.gather(sc, d_hp, d_cp, hf)
            for a, b in zip(back, sh):
                assert np.array_equal(a.values, b.values)
    for d_cp in (1, 2, 4, 8):
        for w in (x for x in range(1, d_cp + 1) if d_cp % x == 0):
            assert np.array_equal(np.array(orc.ring_sources(d_cp, w)), g[f"sched_{d_cp}_{w}"])


def test_zigzag_kats():
    perm, _ = orc.zigzag(8, 2)
    assert set(perm[:4]) == {0, 1, 6, 7} and set(perm[4:]) == {2, 3, 4, 5}
    assert orc.ring_sources(8, 4)[0] == [0, 3, 2, 1, 4, 7, 6, 5]


def test_pipeline_matches_reference():
    g = golden("pipeline_small.npz")
    pos = np.arange(32)
    q, k, v = (orc.Dense(g[n], pos) for n in "qkv")
    for d_hp, d_cp, w in [(1, 1, 1), (2, 2, 2), (4, 2, 1), (8, 2, 2), (1, 8, 4), (2, 4, 4)]:
        for c in (0, 1):
            out = orc.two_d_attention(q, k, v, 8, 2, d_hp, d_cp, w, True, bool(c))
            assert np.max(np.abs(out.values - g[f"out_{d_hp}_{d_cp}_{w}_c{c}"])) <= 1e-12


@pytest.mark.parametrize("name", ["mha_d128_s256_c", "gqa_d128_s384_c",
                                  "mha_d64_s256_n", "gqa_d128_s200_n"])
def test_gpu_fixtures_match_oracle(name):
    g = golden(f"gpu_{name}.npz")
    q, k, v, do = (bf16_bits_to_f64(g[n]) for n in ("q", "k", "v", "do"))
    causal = bool(g["causal"])
    pos = np.arange(q.shape[1])
    out, lse = orc.attention(q, k, v, pos, pos, causal)
    assert np.max(np.abs(out - g["out"])) <= 1e-5
    dq, dk, dv = orc.attention_grads(q, k, v, do, pos, pos, causal)
    for a, b in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        assert np.max(np.abs(a - g[b])) <= 1e-4


def test_gpu_pipeline_fixture_matches_oracle():
    g = golden("gpu_pipeline_c1s.npz")
    pos = np.arange(512)
    q, k, v = (orc.Dense(bf16_bits_to_f64(g[n]), pos) for n in "qkv")
    for hf, name in ((True, "head_first"), (False, "context_first")):
        out = orc.two_d_attention(q, k, v, 8, 8, 2, 2, 2, hf, True)
        assert np.max(np.abs(out.values - g[f"out_{name}"])) <= 1e-5


def test_row_and_key_restricted_grads_match_reference_golden():
    """attention_grads_rows / attention_key_grads (the sampled large-S checks)
    reproduce the reference's own attention_backward output (golden 'big' case,
    causal, S=64) on every row / key subset we slice."""
    g = golden("backward_small.npz")
    q, k, v, do = (g[f"big_{n}"] for n in ("q", "k", "v", "do"))
    pos = np.arange(q.shape[1])
    out, lse = orc.attention(q, k, v, pos, pos, True)
    delta = (do * out).sum(-1)
    rows = np.array([0, 1, 17, 31, 32, 63])
    dq = orc.attention_grads_rows(q, k, v, do[:, rows], pos, pos, rows, True)
    assert np.max(np.abs(dq - g["big_dq"][:, rows])) <= 1e-10
    keys = np.array([0, 5, 31, 62, 63])
    dk, dv = orc.attention_key_grads(q, k, v, do, pos, pos, keys, lse, delta, True)
    assert np.max(np.abs(dk - g["big_dk"][:, keys])) <= 1e-10
    assert np.max(np.abs(dv - g["big_dv"][:, keys])) <= 1e-10


@pytest.mark.parametrize("hkv", [1, 2])
def test_sampled_check_is_exact_on_oracle_outputs(hkv):
    """oracle/sampled.check (blocked f64 row statistics + sampled rows/keys)
    reports ~0 error when fed the dense oracle's own outputs, and its f64 row
    statistics pin to the oracle's LSE / delta."""
    torch = pytest.importorskip("torch")
    from oracle import sampled
    H, S, d = 4, 384, 32
    q, k, v = orc.philox_qkv(5, H, hkv, S, d)
    do = np.random.Generator(np.random.Philox(6)).standard_normal(q.shape)
    pos = np.arange(S)
    out, lse = orc.attention(q, k, v, pos, pos, True)
    dq, dk, dv = orc.attention_grads(q, k, v, do, pos, pos, True)
    T = torch.from_numpy
    res = sampled.check(T(q), T(k), T(v), T(do), T(out), T(dq), T(dk), T(dv), T(lse), causal=True,
                        n_rows=64, n_keys=48, seed=3)
    assert sampled.passes(res, max_abs=1e-10, rel_l2=1e-12, pin=1e-10) == [], res
    assert res["rows"] >= 64 and res["keys"] >= 48
    # a wrong dK column is caught
    dk_bad = dk.copy()
    dk_bad[:, 0] += 0.5
    res = sampled.check(T(q), T(k), T(v), T(do), dk=T(dk_bad), causal=True, n_rows=16, n_keys=16, seed=3)
    assert res["dK"][0] >= 0.49


def test_bf16_round_matches_torch():
    """bf16_round (the kernel precision-policy emulation used by the sampled
    gradient checks) is torch's round-to-nearest-even bf16 conversion."""
    torch = pytest.importorskip("torch")
    x = np.random.Generator(np.random.Philox(9)).standard_normal(100000) * np.exp(
        np.random.Generator(np.random.Philox(10)).uniform(-20, 20, 100000))
    x = np.concatenate([x, [0.0, -0.0, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, 65504.0]])
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).double().numpy()
    assert np.array_equal(orc.bf16_round(x), ref)
