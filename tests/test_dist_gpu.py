"""Multi-GPU parity of the distributed runtime vs the CPU oracle.

Each case launches ``tests/dist_check.py`` under torchrun with one rank per
GPU (skipped when the box has fewer GPUs than the case needs). Tolerance
(bf16 outputs vs the f64 oracle): max-abs <= 2e-2 * max(1, max|ref|) and
rel-L2 <= 1e-2 for O, dQ, dK, dV. The range factor matters only for
gradients whose magnitude exceeds 1 (bf16 keeps 8 mantissa bits).
"""

import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAX_ABS, REL_L2 = 2e-2, 1e-2

CASES = [
    # d_hp, d_cp, w, placement, H, H_kv, S, d
    (2, 1, 1, "head_first", 8, 8, 1024, 128),
    (1, 2, 2, "head_first", 8, 8, 1024, 128),
    (1, 2, 1, "context_first", 4, 2, 1024, 128),
    (2, 2, 2, "head_first", 8, 2, 2048, 128),
    (2, 2, 1, "context_first", 8, 8, 2048, 128),
    (1, 4, 2, "head_first", 4, 4, 2048, 128),
    (1, 4, 4, "context_first", 4, 1, 2048, 128),
    (4, 1, 1, "head_first", 8, 2, 1024, 128),  # GQA replication: H_kv=2 < d_hp=4
    (2, 2, 2, "head_first", 4, 1, 1024, 128),  # replication AND a ring: the fp32 dK/dV home hop
    (2, 2, 2, "context_first", 8, 8, 1024, 64),
    # 8 GPUs (BASELINE configs 3-5 grids at parity sizes)
    (4, 2, 2, "head_first", 8, 8, 2048, 128),
    (4, 2, 1, "context_first", 8, 8, 2048, 128),
    (2, 4, 2, "head_first", 8, 2, 2048, 128),
    (1, 8, 4, "context_first", 4, 4, 2048, 128),
    (8, 1, 1, "head_first", 8, 4, 1024, 128),  # replication: H_kv=4 < d_hp=8
]


def test_dist_non_causal(tmp_path):
    """Full (non-causal) attention through the 2x2 runtime."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    res = _run(4, ["--d-hp", "2", "--d-cp", "2", "--w", "1", "--placement", "head_first", "--heads", "8",
                   "--kv-heads", "4", "--seq", "1024", "--dim", "128", "--causal", "0"], tmp_path)
    for name in ("O", "dQ", "dK", "dV"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"


def _run(nproc, args, tmp_path, env=None, timeout=600):
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "dist_check.py"),
           *args, "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env=None if env is None else {**os.environ, **env})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return json.loads(out.read_text())


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[:3])) + f"-{c[3]}-H{c[4]}-{c[5]}-S{c[6]}-d{c[7]}")
def test_dist_matches_oracle(case, tmp_path):
    d_hp, d_cp, w, pl, H, Hkv, S, d = case
    n = d_hp * d_cp
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    res = _run(n, ["--d-hp", str(d_hp), "--d-cp", str(d_cp), "--w", str(w), "--placement", pl,
                   "--heads", str(H), "--kv-heads", str(Hkv), "--seq", str(S), "--dim", str(d)], tmp_path)
    for name in ("O", "dQ", "dK", "dV"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"


@pytest.mark.parametrize("placement", ["head_first", "context_first"])
def test_dist_golden_config1_shape(placement, tmp_path):
    """Reference run_2d_attention output (golden) at a config-1 shape: H=8 d=64 S=512, 2x2, w=2."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    res = _run(4, ["--d-hp", "2", "--d-cp", "2", "--w", "2", "--placement", placement, "--heads", "8",
                   "--kv-heads", "8", "--seq", "512", "--dim", "64",
                   "--golden", os.path.join(ROOT, "tests", "golden", "gpu_pipeline_c1s.npz")], tmp_path)
    for name in ("O", "O_golden"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"


FUSED = [(2, 2, 2, "head_first", 8, 2, 2048, 128), (1, 2, 1, "context_first", 4, 4, 1024, 128),
         (4, 1, 1, "head_first", 8, 2, 1024, 128), (1, 1, 1, "head_first", 4, 2, 1024, 64)]


@pytest.mark.parametrize("case", FUSED, ids=lambda c: "x".join(map(str, c[:3])) + f"-{c[3]}-H{c[4]}-{c[5]}-d{c[7]}")
def test_dist_token_major_fused_qkv_autograd(case, tmp_path):
    """Token-major strided views of a fused QKV projection output, gradients
    through torch.autograd."""
    d_hp, d_cp, w, pl, H, Hkv, S, d = case
    n = d_hp * d_cp
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    res = _run(n, ["--d-hp", str(d_hp), "--d-cp", str(d_cp), "--w", str(w), "--placement", pl,
                   "--heads", str(H), "--kv-heads", str(Hkv), "--seq", str(S), "--dim", str(d), "--fused-qkv"],
               tmp_path)
    for name in ("O", "dQ", "dK", "dV"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"


SCPP = [(1, 1, 1), (2, 1, 1), (1, 2, 2), (2, 2, 1), (2, 2, 2, "groups")]


@pytest.mark.parametrize("case", SCPP, ids=lambda c: "x".join(map(str, c[:3])) + ("-groups" if len(c) > 3 else ""))
def test_selective_checkpoint_pp(case, tmp_path):
    """SC++ (SURVEY §8f row 2): checkpointed layers recompute everything except
    the whitelisted 2D attention, whose O/LSE are kept — same gradients as plain
    autograd, no attention-forward kernel in the backward pass, while
    torch.utils.checkpoint re-runs the ring forward."""
    d_hp, d_cp, w = case[:3]
    grouped = len(case) > 3  # pipelined head groups (A2D_HEAD_GROUPS=2, GQA 8/4)
    n = d_hp * d_cp
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(ROOT, "tests", "scpp_check.py"),
           "--d-hp", str(d_hp), "--d-cp", str(d_cp), "--w", str(w), "--out", str(out)]
    if grouped:
        cmd += ["--kv-heads", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "A2D_HEAD_GROUPS": "2"} if grouped else None)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for res in json.loads(out.read_text()):
        assert res["grad_rel_l2"] <= 1e-2, res
        assert res["out_max_abs"] == 0.0, res
        k = res["fwd_kernels_in_bwd"]
        assert k["plain"] == 0 and k["scpp"] == 0, res
        assert k["torch_checkpoint"] >= 2 * d_cp, res  # 2 layers x d_cp ring steps recomputed


GROUPED = [
    # d_hp, d_cp, w, placement, H, H_kv, S, d, fused-qkv
    (2, 1, 1, "head_first", 8, 8, 1024, 128, False),
    (2, 2, 2, "head_first", 8, 4, 2048, 128, False),   # GQA inside each head group
    (4, 1, 1, "context_first", 8, 8, 1024, 128, True),  # token-major fused QKV views
    (2, 2, 1, "context_first", 8, 8, 2048, 128, True),
]


@pytest.mark.parametrize("case", GROUPED, ids=lambda c: "x".join(map(str, c[:3])) + f"-{c[3]}-H{c[4]}-{c[5]}"
                         + ("-lhd" if c[8] else ""))
def test_dist_pipelined_head_groups(case, tmp_path):
    """Head-group pipelined exchange (A2D_HEAD_GROUPS=2): group g+1's all-to-all
    overlaps group g's ring; same parity bar as the one-shot exchange."""
    d_hp, d_cp, w, pl, H, Hkv, S, d, fused = case
    n = d_hp * d_cp
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    args = ["--d-hp", str(d_hp), "--d-cp", str(d_cp), "--w", str(w), "--placement", pl,
            "--heads", str(H), "--kv-heads", str(Hkv), "--seq", str(S), "--dim", str(d)]
    res = _run(n, args + (["--fused-qkv"] if fused else []), tmp_path, env={"A2D_HEAD_GROUPS": "2"})
    assert res["head_groups"] == 2
    for name in ("O", "dQ", "dK", "dV"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"


NATIVE = [
    # d_hp, d_cp, w, placement, H, H_kv, S
    (1, 1, 1, "head_first", 4, 2, 1024),
    (2, 1, 1, "head_first", 8, 8, 1024),
    (1, 2, 2, "context_first", 8, 4, 1024),
    (2, 2, 1, "head_first", 8, 8, 2048),
    (1, 4, 2, "head_first", 4, 4, 2048),
    (4, 1, 1, "context_first", 8, 2, 1024),   # GQA replication (H_kv < d_hp)
    (2, 2, 2, "head_first", 4, 1, 1024),      # replication and a ring: fp32 home hop
    (4, 2, 2, "head_first", 8, 8, 2048),      # 8 GPUs: config 3's grid
    (2, 4, 2, "context_first", 8, 2, 2048),   # 8 GPUs: config 4's grid (GQA, w=2)
]


@pytest.mark.parametrize("transport", ["nccl", "symm"])
@pytest.mark.parametrize("case", NATIVE, ids=lambda c: "x".join(map(str, c[:3])) + f"-{c[3]}-H{c[4]}-{c[5]}")
def test_native_runtime_matches_oracle_and_python(case, transport, tmp_path):
    """Native C++ runtime behind the context C ABI: same parity bar
    as the Python runtime, and the same numbers as dist.Attn2D. transport
    "symm": the head-parallel exchange on copy engines into CUDA-IPC-mapped
    peer buffers (d_hp > 1); "nccl": NCCL send/recv."""
    d_hp, d_cp, w, pl, H, Hkv, S = case
    n = d_hp * d_cp
    if transport == "symm" and d_hp == 1:
        pytest.skip("no head-parallel exchange at d_hp = 1")
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    res = _run(n, ["--d-hp", str(d_hp), "--d-cp", str(d_cp), "--w", str(w), "--placement", pl,
                   "--heads", str(H), "--kv-heads", str(Hkv), "--seq", str(S), "--dim", "128", "--native"],
               tmp_path, env={"A2D_TRANSPORT": transport}, timeout=180)
    for name in ("O", "dQ", "dK", "dV"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"
    assert res["native_vs_python"] <= 1e-2, res["native_vs_python"]
    assert res["native_transport"] == transport, res["native_transport"]


@pytest.mark.parametrize("case", [(1, 1, 1, "head_first", 4, 2, 1024), (2, 2, 2, "context_first", 8, 4, 2048)],
                         ids=lambda c: "x".join(map(str, c[:3])) + f"-{c[3]}")
def test_native_two_layers_in_flight(case, tmp_path):
    """Stateless context ABI: layer A's forward, layer B's forward, B's backward,
    then A's backward from A's caller-owned saved state — A still matches the
    oracle (ref ring.py:82-119 is a pure function)."""
    d_hp, d_cp, w, pl, H, Hkv, S = case
    n = d_hp * d_cp
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    res = _run(n, ["--d-hp", str(d_hp), "--d-cp", str(d_cp), "--w", str(w), "--placement", pl,
                   "--heads", str(H), "--kv-heads", str(Hkv), "--seq", str(S), "--dim", "128", "--native",
                   "--two-layers"], tmp_path, timeout=180)
    for name in ("O", "dQ", "dK", "dV"):
        ma, rl, rng = res[name]
        assert ma <= MAX_ABS * max(1.0, rng) and rl <= REL_L2, \
            f"{name}: max-abs {ma:.3e} (range {rng:.2f}) rel-L2 {rl:.3e}"
