"""The reference operator API (paper_2406_18485_b200.api) on the GPU, mirroring
the reference's own tests (pkg/tests/test_oracle.py, test_sharding.py,
test_ring.py) against the golden vectors the reference produced.
Numerics: bf16 kernels vs f64 reference, max-abs <= 2e-2*max(1,|ref|) and
rel-L2 <= 1e-2; layout ops bit-exact."""

import math
import os

import numpy as np
import pytest

from conftest import golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_18485_b200 import api as A
    return A


def close(name, got, ref, tol=2e-2, rel=1e-2):
    got = np.asarray(got.detach().cpu() if isinstance(got, torch.Tensor) else got, np.float64)
    ref = np.asarray(ref, np.float64)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(got), fin), name
    d = np.abs(got[fin] - ref[fin])
    rng = max(1.0, float(np.abs(ref[fin]).max()))
    assert d.max() <= tol * rng and np.linalg.norm(d) <= rel * np.linalg.norm(ref[fin]), \
        f"{name}: max {d.max():.3e} rel {np.linalg.norm(d) / np.linalg.norm(ref[fin]):.3e}"


def bf(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).double().numpy()


def test_full_attention_matches_reference_golden():
    A = api()
    g = golden("attention_small.npz")
    pos = np.arange(16)
    for c in (0, 1):
        q, k, v = (A.DenseTensor(bf(g[f"c{c}_{n}"]), pos) for n in "qkv")
        out, lse = A.full_attention(q, k, v, bool(c))
        close(f"out c{c}", out.values, g[f"c{c}_out"])
        close(f"lse c{c}", lse, g[f"c{c}_lse"])
        assert np.array_equal(out.positions, pos)


def test_permuted_positions_carry_the_mask():
    A = api()
    g = golden("attention_small.npz")
    q = A.DenseTensor(bf(g["perm_q"]), g["perm_pos"])
    k = A.DenseTensor(bf(g["perm_k"]), np.arange(10))
    v = A.DenseTensor(bf(g["perm_v"]), np.arange(10))
    out, _ = A.full_attention(q, k, v, True)
    close("permuted", out.values, g["perm_out"])


def test_block_merge_partitions_and_identities():
    A = api()
    g = golden("merge.npz")
    pos = np.arange(16)
    q = A.DenseTensor(bf(g["q"]), pos)
    for c in (0, 1):
        acc = A.empty_block(4, 16, 8)
        for b in range(4):
            sl = slice(b * 4, (b + 1) * 4)
            blk = A.attention_block(q, A.DenseTensor(bf(g["k"][:, sl]), pos[sl]),
                                    A.DenseTensor(bf(g["v"][:, sl]), pos[sl]), bool(c))
            acc = A.block_update(acc, blk)
        close(f"fold out c{c}", acc.out, g[f"c{c}_acc_out"])
        close(f"fold lse c{c}", acc.lse, g[f"c{c}_acc_lse"])
    blk = A.attention_block(q, A.DenseTensor(bf(g["k"]), pos), A.DenseTensor(bf(g["v"]), pos), False)
    same = A.block_update(A.empty_block(4, 16, 8), blk)
    assert torch.equal(same.out, blk.out) and torch.equal(same.lse, blk.lse)
    twice = A.block_update(blk, blk)
    assert torch.allclose(twice.lse, blk.lse + math.log(2), atol=1e-5)
    assert torch.allclose(twice.out, blk.out, atol=1e-5)


def test_attention_backward_matches_reference_golden():
    A = api()
    g = golden("backward_small.npz")
    pos = np.arange(64)
    q, k, v = (A.DenseTensor(bf(g[f"big_{n}"]), pos) for n in "qkv")
    dq, dk, dv = A.attention_backward(q, k, v, bf(g["big_do"]), True)
    close("dq", dq, g["big_dq"])
    close("dk", dk, g["big_dk"])
    close("dv", dv, g["big_dv"])


@pytest.mark.parametrize("d_hp,d_cp,w", [(1, 1, 1), (2, 2, 2), (4, 2, 1), (8, 2, 2), (1, 8, 4), (2, 4, 4)])
@pytest.mark.parametrize("causal", [0, 1])
def test_run_2d_attention_matches_reference_golden(d_hp, d_cp, w, causal):
    A = api()
    from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig
    g = golden("pipeline_small.npz")
    pos = np.arange(32)
    q, k, v = (A.DenseTensor(bf(g[n]), pos) for n in "qkv")
    model = ModelConfig(seq_len=32, heads=8, kv_heads=2, hidden=32)
    out = A.run_2d_attention(q, k, v, model, ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=w),
                             ClusterConfig(), bool(causal))
    assert np.array_equal(out.positions, pos)
    close("out", out.values, g[f"out_{d_hp}_{d_cp}_{w}_c{causal}"])


def test_run_2d_attention_rejects_invalid_config():
    A = api()
    from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig
    x = A.DenseTensor(np.zeros((4, 12, 8)), np.arange(12))
    with pytest.raises(ValueError, match="invalid configuration"):
        A.run_2d_attention(x, x, x, ModelConfig(12, 4, 4, 32), ParallelConfig(d_hp=3, d_cp=1),
                           ClusterConfig(), True)


def test_seq_alltoall_bit_exact_on_gpu():
    A = api()
    from paper_2406_18485_b200.config import ClusterConfig, ParallelConfig, Placement, build_rank_grid
    g = golden("layouts.npz")
    vals = np.arange(8 * 64 * 2, dtype=np.float64).reshape(8, 64, 2)
    x = A.DenseTensor(torch.from_numpy(vals).to(torch.float32).cuda(), np.arange(64))
    for d_hp, d_cp in ((2, 2), (4, 2), (2, 4), (8, 1)):
        for pl in Placement:
            grid = build_rank_grid(ParallelConfig(d_hp=d_hp, d_cp=d_cp, placement=pl), ClusterConfig())
            sh = A.shard_sequence(x, grid)
            sc = A.seq_alltoall_scatter(sh, grid)
            tag = f"{d_hp}x{d_cp}_{pl.value}"
            got = np.stack([c.values.cpu().numpy() for c in sc.chunks])
            assert np.array_equal(got, g[f"headvals_{tag}"]), tag
            assert np.array_equal(np.stack([c.positions for c in sc.chunks]), g[f"headpos_{tag}"])
            back = A.seq_alltoall_gather(sc, grid)
            for a, b in zip(back.chunks, sh.chunks):
                assert torch.equal(a.values, b.values)
            assert torch.equal(A.unshard(back).values, x.values)


def test_kv_replicate_contiguous_copies():
    A = api()
    from paper_2406_18485_b200.config import ClusterConfig, ParallelConfig, build_rank_grid
    grid = build_rank_grid(ParallelConfig(d_hp=16, d_cp=1), ClusterConfig())
    kv = A.shard_sequence(A.DenseTensor(torch.randn(8, 32, 2).cuda(), np.arange(32)), grid)
    rep = A.kv_replicate(kv, 8, 16, 32)
    c = rep.chunks[0].values
    assert c.shape[0] == 16
    for h in range(8):
        assert torch.equal(c[2 * h], c[2 * h + 1])
    with pytest.raises(ValueError):
        A.kv_replicate(kv, 8, 64, 32)


def test_verify_cli_lattice_and_fault_injection():
    """tests/verify_cli.py mirrors the reference's `attn2d verify` (cli.py:46-122):
    the whole lattice passes (exit 0), --inject-fault is detected (exit 1),
    a bad S / d_sp combination is a config error (exit 2)."""
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cli = [sys.executable, os.path.join(root, "tests", "verify_cli.py")]
    r = subprocess.run(cli, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "OK: all" in r.stdout
    n = sum(1 for line in r.stdout.splitlines() if "max|delta|" in line)
    assert n == 304  # the reference verify lattice (cli.py:58-91): 2 H_kv x 2 S x 2 causal x 38 grids
    r = subprocess.run(cli + ["--acceptance"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    n = sum(1 for line in r.stdout.splitlines() if "max|delta|" in line)
    assert n > 500  # acceptance criterion 1's lattice (test_acceptance.py:53-91)
    r = subprocess.run(cli + ["--seq", "32", "--inject-fault"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 1 and "FAIL" in r.stdout
    r = subprocess.run(cli + ["--seq", "36", "--dsp", "4"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2
