"""B200-calibrated step-time model and planner for 2D-Attention.

The reference ranks (d_hp, d_cp, w, placement) with A100-era closed forms
(`/root/reference/pkg/src/attn2d/costs.py:171-206`, `planner.py:39-112`). This
module keeps the same enumeration rule but predicts the step time of THIS
implementation from constants measured on B200 (kernel throughput per chunk
kernel, NVLink all-to-all / point-to-point bandwidth) and from how the runtime
overlaps communication (`dist.Attn2D`): the head-parallel all-to-alls are on the
critical path; a ring hop overlaps the attention step it runs beside, so only
max(0, t_hop - t_step) is exposed; the backward dK/dV accumulator hop (fp32,
twice the KV bytes) is exposed for its remainder after the next step's compute
and its K4 add is HBM time.

`calibration()` returns the measured defaults; `check_against_sweep()` compares
predictions with `profiles/r01_sweep_*.jsonl` (tests pin the ranking quality).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

from .config import ClusterConfig, ModelConfig, ParallelConfig, Placement, replicated_kv_heads, validate


@dataclass(frozen=True)
class B200Calibration:
    """Measured on B200 (round 1): tools/kbench.py, bench.py sweeps, tools/trace.py
    phase traces (profiles/r01_trace_*.json), guide peaks."""

    fwd_tflops: float = 1310.0     # forward chunk kernel in a full step (final round-2b build: P in quarters)
    bwd_tflops: float = 1135.0     # backward chunk kernel in a full step (128-query kernel, CTA pairs)
    short_chunk_tokens: float = 500.0   # kernel efficiency ~ C / (C + this) for small chunks
    a2a_gbs: float = 620.0         # NCCL all_to_all_single: time ~ whole buffer / this (traces, d_hp = 2 and 4)
    ce_gbs: float = 770.0          # copy-engine write into a peer's symmetric buffer (tools/probes/peer_probe.py)
    transport: str = "symm"        # dist.Attn2D default; "nccl" for the round-1 sweeps
    p2p_gbs: float = 770.0         # per-direction peer bandwidth (B200 profiling guide)
    hbm_gbs: float = 6527.5        # MEASURED_PEAKS hbm_gbs (K4 add)
    pack_gbs: float = 5500.0       # achieved by the pack / permute / convert kernels (traces)
    ring_overhead: float = 0.045   # d_cp > 1: ring-step compute slowdown (per-step merge / K4 traffic,
                                   # smaller chunks, NCCL copy kernels sharing SMs) — sweeps and traces
    launch_s: float = 12e-6        # per NCCL call / kernel launch overhead
    elem: int = 2                  # bf16


def calibration() -> B200Calibration:
    return B200Calibration()


# The earlier round-1 build that produced profiles/r01_sweep_*.jsonl (NCCL
# all-to-all, backward before the transposed-dQ drain).
EARLY_ROUND1 = B200Calibration(fwd_tflops=1100.0, bwd_tflops=940.0, transport="nccl")
# The final round-1 / round-2 builds (64-query backward) that produced
# profiles/r01_final_sweep_S128k_symm_2_4gpu.jsonl.
ROUND2 = B200Calibration(fwd_tflops=1180.0, bwd_tflops=1040.0)
# The first round-2b build (128-query backward without pairs, forward P
# released once) that produced profiles/r02b_sweep_S128k_4gpu.jsonl.
ROUND2B_SWEEP = B200Calibration(fwd_tflops=1195.0, bwd_tflops=1110.0)


def _eff(c: B200Calibration, tokens: int) -> float:
    return tokens / (tokens + c.short_chunk_tokens)


def predict(model: ModelConfig, par: ParallelConfig, cal: B200Calibration | None = None,
            causal: bool = True) -> dict:
    """Predicted per-step (fwd+bwd) times in seconds for one layer."""
    cal = cal or calibration()
    S, H, Hkv, d = model.seq_len, model.heads, model.kv_heads, model.head_dim
    d_hp, d_cp, w = par.d_hp, par.d_cp, par.inner_ring
    d_sp = d_hp * d_cp
    Hrep = replicated_kv_heads(Hkv, d_hp, H)
    C, L = S // d_cp, S // d_sp
    frac = 0.5 if causal else 1.0
    flops = 4.0 * S * S * H * d * frac / d_sp           # forward FLOPs per GPU
    eff = _eff(cal, C)
    ring = 1.0 + (cal.ring_overhead if d_cp > 1 else 0.0)
    t_fwd = ring * flops / (cal.fwd_tflops * 1e12 * eff)
    t_bwd = ring * 2.5 * flops / (cal.bwd_tflops * 1e12 * eff)
    # head-parallel exchange phases (critical path), as implemented in dist.Attn2D:
    # fwd in q,k,v / out O, bwd in dO / out dQ,dK,dV (fp32 -> bf16 fused into the pack)
    Tq = H * L * d * cal.elem               # bytes of one (H, L, d) bf16 tensor per rank
    Tkv = 2 * Hrep * L * d * cal.elem       # k and v after replication
    hbm = lambda b: b / (cal.pack_gbs * 1e9)  # noqa: E731
    if d_hp > 1:
        if cal.transport == "nccl":
            net = lambda b: b / (cal.a2a_gbs * 1e9) + cal.launch_s  # noqa: E731
        else:  # crossing bytes on the copy engines + the local chunk copy + a device barrier
            net = lambda b: (b * (d_hp - 1) / d_hp / (cal.ce_gbs * 1e9) + hbm(2 * b / d_hp)  # noqa: E731
                             + 2 * cal.launch_s)
        t_fwd_in = net(Tq) + net(Tkv) + hbm(2 * Tkv + 2 * (Tq + Tkv))   # kv pack, unpack permutes
        t_fwd_out = net(Tq) + hbm(2 * Tq)
        t_bwd_in = net(Tq) + hbm(2 * Tq)
        t_bwd_out = net(Tq) + net(Tkv) + hbm(3 * (Tq + Tkv))
    else:
        t_fwd_in, t_fwd_out, t_bwd_in = hbm(2 * Tkv), hbm(2 * Tq), 0.0
        t_bwd_out = hbm(3 * (Tq + Tkv))
    t_a2a = t_fwd_in + t_fwd_out + t_bwd_in + t_bwd_out
    # ring hops: d_cp - 1 KV hops per pass, each beside one attention step
    kv_bytes = 2 * (Hrep // d_hp) * C * d * cal.elem
    t_hop = kv_bytes / (cal.p2p_gbs * 1e9) + cal.launch_s
    step_f, step_b = t_fwd / d_cp, t_bwd / d_cp
    n_outer = d_cp // w
    exposed = 0.0
    if d_cp > 1:
        # inner hops overlap one step; an outer hop is issued at the start of its
        # outer step and overlaps all w micro-steps of it
        inner_hops = (w - 1) * n_outer
        outer_hops = n_outer - 1
        for step in (step_f, step_b):
            exposed += inner_hops * max(0.0, t_hop - step) + outer_hops * max(0.0, t_hop - w * step)
        # backward dK/dV accumulator (fp32 = 2x bytes) hop after every step + K4 add
        t_dkv = 2 * kv_bytes / (cal.p2p_gbs * 1e9) + cal.launch_s
        exposed += (d_cp - 1) * max(0.0, t_dkv - step_b) + t_dkv  # the home hop is exposed
        exposed += d_cp * (3 * 2 * kv_bytes) / (cal.hbm_gbs * 1e9)
    t = t_fwd + t_bwd + t_a2a + exposed
    total = 3.5 * 4.0 * S * S * H * d * frac  # algorithmic fwd+bwd FLOPs of the layer
    return {"t_step": t, "t_fwd": t_fwd, "t_bwd": t_bwd, "t_a2a": t_a2a, "t_ring_exposed": exposed,
            "t_phases": {"fwd.a2a_in": t_fwd_in, "fwd.a2a_out": t_fwd_out, "bwd.a2a_in": t_bwd_in,
                         "bwd.a2a_out": t_bwd_out},
            "tflops_per_gpu": total / d_sp / t / 1e12, "total_tflops": total / t / 1e12}


def enumerate_configs(model: ModelConfig, n_gpus: int, cluster: ClusterConfig | None = None):
    """Every valid (d_hp, d_cp, w, placement) with d_hp * d_cp = n_gpus
    (same rule as the reference, planner.py:39-59)."""
    cluster = cluster or ClusterConfig()
    out = []
    for d_hp in range(1, n_gpus + 1):
        if n_gpus % d_hp:
            continue
        d_cp = n_gpus // d_hp
        for w in range(1, d_cp + 1):
            if d_cp % w:
                continue
            for pl in Placement:
                par = ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=w, placement=pl)
                if validate(model, par, cluster).ok:
                    try:
                        replicated_kv_heads(model.kv_heads, d_hp, model.heads)
                    except ValueError:
                        continue
                    if replicated_kv_heads(model.kv_heads, d_hp, model.heads) % d_hp:
                        continue
                    out.append(par)
    return out


def plan(model: ModelConfig, n_gpus: int, cal: B200Calibration | None = None, causal: bool = True):
    """Configurations ranked by predicted step time (fastest first)."""
    rows = [(predict(model, p, cal, causal)["t_step"], p) for p in enumerate_configs(model, n_gpus)]
    rows.sort(key=lambda r: (r[0], r[1].d_hp, r[1].inner_ring, r[1].placement.value))
    return rows


def check_against_sweep(path: str, cal: B200Calibration | None = None) -> dict:
    """Compare predictions with a measured sweep (tools/sweep.py JSONL; the
    round-1 sweeps ran the NCCL transport)."""
    cal = cal or calibration()
    errs, pairs = [], []
    for line in open(path):
        r = json.loads(line)
        if r.get("value") is None:
            continue
        s = r["sweep"]
        model = ModelConfig(seq_len=s["seq"], heads=32, kv_heads=32, hidden=32 * 128)
        par = ParallelConfig(d_hp=s["d_hp"], d_cp=s["d_cp"], inner_ring=s["w"], placement=Placement(s["placement"]))
        t_pred = predict(model, par, cal)["t_step"]
        t_meas = r["ms_per_step"] * 1e-3
        errs.append(abs(t_pred - t_meas) / t_meas)
        pairs.append((s["n"], t_pred, t_meas))
    return {"n": len(errs), "mean_rel_err": sum(errs) / max(1, len(errs)), "max_rel_err": max(errs, default=math.nan),
            "pairs": pairs}
