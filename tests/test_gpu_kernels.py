"""Single-GPU parity of the sm_100a kernels against the CPU oracle and the
reference's golden vectors. Tolerances (BASELINE.json north star): bf16
kernels vs the f64 oracle, max-abs <= 2e-2 * max(1, max|ref|) and rel-L2 <=
1e-2 (O, LSE, dQ, dK, dV); permutations bit-exact."""

import math

import numpy as np
import pytest

from conftest import bf16_bits_to_f64, golden
from oracle import attn2d_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
REL_L2 = 1e-2


def close(name, got, ref, max_abs=MAX_ABS, rel=REL_L2):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(got), fin), f"{name}: finiteness pattern differs"
    if not fin.any():
        return
    d = np.abs(got[fin] - ref[fin])
    ma = float(d.max())
    rl = float(np.linalg.norm(d) / max(np.linalg.norm(ref[fin]), 1e-30))
    rng = float(np.abs(ref[fin]).max())
    assert ma <= max_abs * max(1.0, rng) and rl <= rel, f"{name}: max-abs {ma:.3e} (range {rng:.2f}), rel-L2 {rl:.3e}"


def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def t_bf16(bits, device):
    x = torch.from_numpy(np.asarray(bits, np.uint16).view(np.int16).copy())
    return x.view(torch.bfloat16).to(device)


def bf16_round(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def test_umma_selftest():
    from paper_2406_18485_b200 import kernels as K
    d = dev()
    g = torch.Generator().manual_seed(0)
    a, b, v, at = (torch.randn(128, 128, generator=g).to(torch.bfloat16).to(d) for _ in range(4))
    c = K.selftest_umma(a, b, v, at).cpu().double()
    A, B, V, AT = (x.double().cpu() for x in (a, b, v, at))
    refs = [A @ B.T, A @ V, AT.T @ B.T, A @ V]
    for i, r in enumerate(refs):
        err = (c[i] - r).abs().max().item()
        assert err < 1e-2 * max(1.0, r.abs().max().item() / 10), f"case {i}: max err {err}"


def _fwd(q, k, v, q_pos, k_pos, causal, device, scale=None):
    from paper_2406_18485_b200 import kernels as K
    d = q.shape[-1]
    dk = K.fwd_dim(d)
    qt, kt, vt = (K.pad_dim(torch.from_numpy(np.asarray(x, np.float32)).to(device), dk) for x in (q, k, v))
    qp = K.ChunkPlan(torch.as_tensor(q_pos, dtype=torch.int32, device=device))
    kp = K.ChunkPlan(torch.as_tensor(k_pos, dtype=torch.int32, device=device))
    H, T = q.shape[0], q.shape[1]
    lse = torch.empty((H, T), dtype=torch.float32, device=device)
    acc = torch.empty((H, T, dk), dtype=torch.float32, device=device)
    out = torch.empty((H, T, dk), dtype=torch.bfloat16, device=device)
    K.fwd_chunk(qt, kt, vt, qp, kp, causal, scale or 1.0 / math.sqrt(d), lse, acc, out)
    torch.cuda.synchronize()
    return acc[..., :d].cpu().numpy(), lse.cpu().numpy(), out[..., :d].float().cpu().numpy()


@pytest.mark.parametrize("name", ["mha_d128_s256_c", "gqa_d128_s384_c", "mha_d64_s256_n", "gqa_d128_s200_n"])
def test_fwd_chunk_golden(name):
    d = dev()
    g = golden(f"gpu_{name}.npz")
    q, k, v = (bf16_bits_to_f64(g[n]) for n in "qkv")
    pos = np.arange(q.shape[1])
    o, lse, ob = _fwd(q, k, v, pos, pos, bool(g["causal"]), d)
    close(f"{name} O", o, g["out"])
    close(f"{name} O(bf16)", ob, g["out"])
    close(f"{name} LSE", lse, g["lse"])


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", [(4, 4, 1024, 128), (8, 2, 640, 128), (2, 1, 300, 64), (2, 2, 7, 128)])
def test_fwd_chunk_oracle(shape, causal):
    d = dev()
    H, Hkv, T, D = shape
    q, k, v = (bf16_round(x) for x in orc.philox_qkv(31, H, Hkv, T, D))
    pos = np.arange(T)
    o, lse, _ = _fwd(q, k, v, pos, pos, causal, d)
    ro, rl = orc.attention(q, k, v, pos, pos, causal)
    close("O", o, ro)
    close("LSE", lse, rl)


@pytest.mark.parametrize("d_cp", [2, 4])
def test_fwd_zigzag_steps_and_merge(d_cp):
    """Every (Q chunk j, KV chunk s) pair of a zig-zag ring, folded with the
    fused merge, equals full attention (ref run_double_ring)."""
    from paper_2406_18485_b200 import kernels as K
    d = dev()
    H, S, D = 2, 1024, 128
    q, k, v = (bf16_round(x) for x in orc.philox_qkv(5, H, H, S, D))
    perm, _ = orc.zigzag(S, d_cp)
    C = S // d_cp
    ro, rl = orc.attention(q, k, v, np.arange(S), np.arange(S), True)
    for j in range(d_cp):
        qpos = perm[j * C:(j + 1) * C]
        qt = K.pad_dim(torch.from_numpy(q[:, qpos].astype(np.float32)).to(d), 128)
        qp = K.ChunkPlan(torch.as_tensor(qpos, dtype=torch.int32, device=d))
        lse = torch.empty((H, C), dtype=torch.float32, device=d)
        acc = torch.empty((H, C, 128), dtype=torch.float32, device=d)
        for step, s in enumerate(orc.ring_sources(d_cp, d_cp)[j]):
            kpos = perm[s * C:(s + 1) * C]
            kt = K.pad_dim(torch.from_numpy(k[:, kpos].astype(np.float32)).to(d), 128)
            vt = K.pad_dim(torch.from_numpy(v[:, kpos].astype(np.float32)).to(d), 128)
            kp = K.ChunkPlan(torch.as_tensor(kpos, dtype=torch.int32, device=d))
            K.fwd_chunk(qt, kt, vt, qp, kp, True, 1 / math.sqrt(D), lse, acc, None, merge=step > 0)
        torch.cuda.synchronize()
        close(f"rank {j} O", acc.cpu().numpy(), ro[:, qpos])
        close(f"rank {j} LSE", lse.cpu().numpy(), rl[:, qpos])


def _bwd(q, k, v, do, q_pos, k_pos, causal, device, bd=None):
    """Forward then backward chunk; the backward runs at head dim bd (default:
    the forward's 64 / 128 kernel dim, i.e. the d=64 kernel for d <= 64)."""
    from paper_2406_18485_b200 import kernels as K
    D = q.shape[-1]
    fd = K.fwd_dim(D)
    bd = bd or fd
    H, T = q.shape[0], q.shape[1]
    Hkv, Tk = k.shape[0], k.shape[1]
    t = lambda x, dd: K.pad_dim(torch.from_numpy(np.asarray(x, np.float32)).to(device), dd)  # noqa: E731
    qp = K.ChunkPlan(torch.as_tensor(q_pos, dtype=torch.int32, device=device))
    kp = K.ChunkPlan(torch.as_tensor(k_pos, dtype=torch.int32, device=device))
    scale = 1 / math.sqrt(D)
    lse = torch.empty((H, T), dtype=torch.float32, device=device)
    out = torch.empty((H, T, fd), dtype=torch.bfloat16, device=device)
    K.fwd_chunk(t(q, fd), t(k, fd), t(v, fd), qp, kp, causal, scale, lse, None, out)
    dot = t(do, fd)
    lse2, delta = K.bwd_preprocess(out, dot, lse)
    dq_acc = K.dq_acc_t(H, T, device, bd)
    dk = torch.empty((Hkv, Tk, bd), dtype=torch.float32, device=device)
    dv = torch.empty((Hkv, Tk, bd), dtype=torch.float32, device=device)
    K.bwd_chunk(t(q, bd), t(k, bd), t(v, bd), t(do, bd), qp, kp, lse2, delta, dq_acc, dk, dv, False,
                causal, scale)
    torch.cuda.synchronize()
    dq = K.dq_from_acc(dq_acc, T)
    return (dq[..., :D].cpu().numpy(), dk[..., :D].cpu().numpy(), dv[..., :D].cpu().numpy())


@pytest.mark.parametrize("name", ["mha_d128_s256_c", "gqa_d128_s384_c", "mha_d64_s256_n", "gqa_d128_s200_n"])
def test_bwd_chunk_golden(name):
    d = dev()
    g = golden(f"gpu_{name}.npz")
    q, k, v, do = (bf16_bits_to_f64(g[n]) for n in ("q", "k", "v", "do"))
    pos = np.arange(q.shape[1])
    dq, dk, dv = _bwd(q, k, v, do, pos, pos, bool(g["causal"]), d)
    close(f"{name} dQ", dq, g["dq"])
    close(f"{name} dK", dk, g["dk"])
    close(f"{name} dV", dv, g["dv"])


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", [(4, 2, 768, 128), (2, 2, 130, 128), (4, 2, 768, 64), (2, 1, 333, 64),
                                   (2, 2, 200, 48)])
def test_bwd_chunk_oracle(shape, causal):
    d = dev()
    H, Hkv, T, D = shape
    q, k, v = (bf16_round(x) for x in orc.philox_qkv(77, H, Hkv, T, D))
    do = bf16_round(np.random.Generator(np.random.Philox(78)).standard_normal(q.shape))
    pos = np.arange(T)
    dq, dk, dv = _bwd(q, k, v, do, pos, pos, causal, d)
    rq, rk, rv = orc.attention_grads(q, k, v, do, pos, pos, causal)
    close("dQ", dq, rq)
    close("dK", dk, rk)
    close("dV", dv, rv)


def test_bwd_d64_kernel_matches_padded_d128():
    """The D=64 backward instantiation (BASELINE config 1's head dim) against
    the same gradients from the zero-padded D=128 kernel and the oracle."""
    d = dev()
    H, Hkv, T, D = 4, 2, 640, 64
    q, k, v = (bf16_round(x) for x in orc.philox_qkv(5, H, Hkv, T, D))
    do = bf16_round(np.random.Generator(np.random.Philox(6)).standard_normal(q.shape))
    pos = np.arange(T)
    g64 = _bwd(q, k, v, do, pos, pos, True, d)
    g128 = _bwd(q, k, v, do, pos, pos, True, d, bd=128)
    ref = orc.attention_grads(q, k, v, do, pos, pos, True)
    for name, a, b, r in zip(("dQ", "dK", "dV"), g64, g128, ref):
        close(name + " d64", a, r)
        assert np.max(np.abs(a - b)) <= 1e-3 * max(1.0, np.abs(r).max()), name


def test_permute_and_gather_bit_exact():
    from paper_2406_18485_b200 import kernels as K
    d = dev()
    x = torch.randint(-2**15, 2**15, (4, 3, 40, 16), dtype=torch.int16, device=d).view(torch.bfloat16)
    y = K.permute_blocks(x, 4, 3).view(3, 4, 40, 16)
    assert torch.equal(y.view(torch.int16), x.view(torch.int16).permute(1, 0, 2, 3).contiguous())
    idx = torch.tensor([2, 0, 0, 1, 3, 3], dtype=torch.int32, device=d)
    out = torch.empty((6, 3, 40, 16), dtype=torch.bfloat16, device=d)
    K.gather_blocks(x, idx, out)
    assert torch.equal(out.view(torch.int16), x.view(torch.int16)[idx.long()])


def test_permute_f32_to_bf16_matches_torch_rounding():
    """Gradient-gather pack: fp32 -> bf16 (round to nearest even) fused with the
    [A][B] -> [B][A] block permute; bit-exact vs torch, incl. A = B = 1."""
    from paper_2406_18485_b200 import kernels as K
    d = dev()
    x = torch.randn(4, 3, 40, 16, device=d) * 100
    y = K.permute_to_bf16(x, 4, 3).view(3, 4, 40, 16)
    assert torch.equal(y.view(torch.int16), x.permute(1, 0, 2, 3).contiguous().bfloat16().view(torch.int16))
    z = K.permute_to_bf16(x, 1, 1)
    assert torch.equal(z.view(torch.int16), x.bfloat16().view(torch.int16))
    with pytest.raises(ValueError):
        K.permute_to_bf16(torch.zeros(3, 2, 5, device=d), 3, 2)  # block of 5 values: not a multiple of 8


@pytest.mark.parametrize("T,A", [(200, 1), (256, 2), (96, 4)])
def test_dqt_to_bf16_transposes_and_packs(T, A):
    """Transposed dQ accumulator [H][128][T_pad] -> bf16 [A][H][T/A][128]
    (peer-major pack when A = d_hp); bit-exact vs torch's rounding."""
    from paper_2406_18485_b200 import kernels as K
    d = dev()
    H = 3
    acc = torch.randn(H, 128, (T + 63) // 64 * 64, device=d) * 10
    out = K.dqt_to_bf16(acc, T, A)
    ref = acc[:, :, :T].transpose(1, 2).reshape(H, A, T // A, 128).transpose(0, 1).contiguous().bfloat16()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def test_bwd_query_slicing_beyond_one_launch():
    """Query chunks longer than one launch's live list (4096 tiles = 262144
    rows) run as consecutive slices; dK/dV must still sum over all of them."""
    d = dev()
    H, Hkv, Tq, Tk, D = 2, 1, 262144 + 130, 200, 128
    rng = np.random.Generator(np.random.Philox(91))
    q = bf16_round(rng.standard_normal((H, Tq, D)) * 0.5)
    k = bf16_round(rng.standard_normal((Hkv, Tk, D)) * 0.5)
    v = bf16_round(rng.standard_normal((Hkv, Tk, D)))
    do = bf16_round(rng.standard_normal((H, Tq, D)))
    qpos, kpos = np.arange(Tq) + 1000, np.arange(Tk)   # every query sees every key (causal, full tiles)
    dq, dk, dv = _bwd(q, k, v, do, qpos, kpos, True, d)
    rows = np.concatenate([np.arange(0, 64), np.arange(262100, Tq)])
    rq, rk, rv = orc.attention_grads(q, k, v, do, qpos, kpos, True)
    close("dQ (sampled rows)", dq[:, rows], rq[:, rows])
    close("dK", dk, rk)
    close("dV", dv, rv)


def test_gather_tokens_bit_exact_and_shard_roundtrip():
    """a2d_gather_tokens (data-loader shard of ref shard_sequence / unshard,
    sharding.py:56-106): gather and scatter are bit-exact byte moves, and the
    global-view shard -> unshard through it is the identity for bf16 d=128."""
    from paper_2406_18485_b200 import api
    from paper_2406_18485_b200 import kernels as K
    from paper_2406_18485_b200.config import ClusterConfig, ParallelConfig, Placement, build_rank_grid
    d = dev()
    x = torch.randint(-2**15, 2**15, (3, 96, 128), dtype=torch.int16, device=d).view(torch.bfloat16)
    idx = torch.randperm(96, device=d)[:40]
    got = K.gather_tokens(x, idx)
    assert torch.equal(got.view(torch.int16), x.view(torch.int16)[:, idx.long()])
    back = torch.zeros_like(x)
    K.gather_tokens(got, idx, out=back, scatter=True)
    ref = torch.zeros_like(x)
    ref[:, idx.long()] = x[:, idx.long()]
    assert torch.equal(back.view(torch.int16), ref.view(torch.int16))
    S = 256
    vals = torch.randn(4, S, 128, device=d).to(torch.bfloat16)
    pos = np.arange(S)
    for d_hp, d_cp in ((2, 2), (1, 4), (4, 1)):
        for pl in Placement:
            grid = build_rank_grid(ParallelConfig(d_hp=d_hp, d_cp=d_cp, placement=pl), ClusterConfig())
            sh = api.shard_sequence(api.DenseTensor(vals, pos), grid)
            perm, _ = orc.zigzag(S, d_cp)
            for j in range(d_cp):
                for i in range(d_hp):
                    c = sh.chunk(i, j)
                    L = S // (d_hp * d_cp)
                    want = perm[j * (S // d_cp) + i * L: j * (S // d_cp) + (i + 1) * L]
                    assert np.array_equal(c.positions, want)
                    assert torch.equal(c.values, vals[:, torch.as_tensor(want, device=d)])
            assert torch.equal(api.unshard(sh).values, vals)
