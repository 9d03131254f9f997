"""2D-Attention fwd+bwd throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

One step = one 2D-Attention layer forward + backward on the global sequence
(S=131072, H=32, d=128, MHA, causal — BASELINE config 3's shape) through the
SPMD runtime (``paper_2406_18485_b200.dist.Attn2D``): HP all-to-all, Double-
Ring attention, all-to-all back, then the backward ring. Inputs are random
bf16 (synthetic; the path has no weights). Algorithmic FLOPs per step:
7 * S^2 * H * d (causal fwd 2 S^2 H d + bwd 2.5x), counted on query heads.

`value` is whole-job TFLOP/s with inputs resident in HBM; `e2e` repeats the
step through the same public API with the step's inputs copied from pinned
host memory and its gradients (dq, dk, dv) copied back inside the timed
region. Rank 0 prints one JSON line.
"""

from __future__ import annotations

import os as _os
import sys as _sys

if "reference" in _sys.argv:  # CPU arm: undo torchrun's OMP_NUM_THREADS=1 before numpy loads its BLAS
    _n = str(len(_os.sched_getaffinity(0)) if hasattr(_os, "sched_getaffinity") else (_os.cpu_count() or 1))
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        _os.environ[_v] = _n

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2D-Attention fwd+bwd TFLOP/s/GPU (MFU) at S=128K, 1/2/4/8 B200"
UNIT = "TFLOP/s"


def default_grid(n: int):
    """(d_hp, d_cp, w) per GPU count. N=2, 4: the fastest factorisation of the
    measured S=128K sweep (profiles/r02_final_sweep_S128k_2_4gpu.jsonl; also the
    planner's pick, tools/plan.py); N=8: BASELINE config 3's 4x2 grid, inner
    ring w=1 (w=1 beat w=2 by 1.7% at 2x2 in the same sweep)."""
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (4, 1, 1), 8: (4, 2, 1)}.get(n, (n, 1, 1))


def peaks():
    p = {"hbm_gbs": 6527.5, "bf16_tflops": 1665.8, "bf16_tflops_sustained": 1389.6, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["src"] = "measured"
    except OSError:
        pass
    return p


# --------------------------------------------------------------------- clocks
REASONS = ["clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
           "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = "index,clocks.sm,clocks.max.sm,power.draw," + ",".join(REASONS)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 4 + len(REASONS):
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for name, val in zip(REASONS, parts[4:]):
                    if val.lower() == "active":
                        reasons.add(name.split(".")[-1])
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU leg
def cpu_sample(rows: int, S: int, d: int, seed: int = 0):
    """Oracle port (oracle/attn2d_oracle.py, f64 numpy/BLAS) on a bounded sample
    of the workload: 1 head x the last `rows` query positions x all S keys,
    fwd + bwd. Returns (seconds, algorithmic FLOPs of the sample)."""
    import numpy as np

    from oracle import attn2d_oracle as orc

    rng = np.random.Generator(np.random.Philox(seed))
    q = rng.standard_normal((1, rows, d))
    k = rng.standard_normal((1, S, d))
    v = rng.standard_normal((1, S, d))
    do = rng.standard_normal((1, rows, d))
    qpos = np.arange(S - rows, S)
    kpos = np.arange(S)
    t0 = time.perf_counter()
    orc.attention(q, k, v, qpos, kpos, True)
    orc.attention_grads(q, k, v, do, qpos, kpos, True)
    dt = time.perf_counter() - t0
    admitted = float(sum(int(p) + 1 for p in qpos))  # causal (query, key) pairs
    flops = 3.5 * 4.0 * admitted * d
    return dt, flops


class all_blas_threads:
    """Use every core this process may run on for the numpy/BLAS CPU legs
    (torchrun sets OMP_NUM_THREADS=1, which would silently cap them at one)."""

    def __enter__(self):
        try:
            from threadpoolctl import threadpool_limits
            n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
            self._ctl = threadpool_limits(limits=n, user_api="blas")
        except Exception:
            self._ctl = None
        return self

    def __exit__(self, *exc):
        if self._ctl is not None:
            self._ctl.restore_original_limits()
        return False


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        n = max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
        return int(n)
    except Exception:
        return os.cpu_count() or 1


def grid_of(a, world: int):
    """(d_hp, d_cp, w) of this run: flags, else default_grid(world)."""
    d_hp, d_cp, w = default_grid(world)
    d_hp, d_cp = a.d_hp or d_hp, a.d_cp or d_cp
    w = a.w or (w if (a.d_hp == 0 and a.d_cp == 0) else d_cp)
    return d_hp, d_cp, w


def workload_config(a, world: int) -> dict:
    """The `config` object both arms print (same workload, same grid)."""
    d_hp, d_cp, w = grid_of(a, world)
    return {"workload": f"2D-Attention fwd+bwd MHA H={a.heads} H_kv={a.kv_heads} D={a.dim} S={a.seq} causal",
            "d_hp": d_hp, "d_cp": d_cp, "w": w, "placement": a.placement, "global_tokens": a.seq,
            "l2": "inputs > L2 (each q/k/v tensor >= 128 MiB per rank), no flush"}


def run_reference(a, rank: int, world: int):
    """--impl reference: the reference's CPU algorithm (oracle port) on host cores."""
    if rank != 0:
        return 0
    S, H, d = a.seq, a.heads, a.dim
    rows = a.cpu_rows
    times, flops = [], 0.0
    with all_blas_threads():
        for _ in range(a.warmup if a.warmup < 1 else 1):
            cpu_sample(64, S, d)
        for _ in range(a.steps):
            dt, fl = cpu_sample(rows, S, d)
            times.append(dt)
            flops = fl
        cores = cpu_cores()
    tot = sum(times)
    val = flops * len(times) / tot / 1e12
    sample = f"1 head x last {rows} query rows x {S} keys, d={d}, causal fwd+bwd, f64 numpy (oracle port)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": tot / len(times) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(a, world),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


HBM_KERNELS = ("a2d_bwd_preprocess", "a2d_dqt_to_bf16", "a2d_dqt_to_bf16_d", "a2d_permute_blocks", "a2d_gather_blocks",
               "a2d_permute_f32_to_bf16", "a2d_copy_rows", "a2d_merge", "a2d_add_f32", "a2d_f32_to_bf16",
               "a2d_sum_replicas_f32")


def hbm_roofline(events, peak_gbs: float) -> dict:
    """Per HBM-bound kernel: algorithmic bytes (read + write of every element
    moved, from the wrappers in kernels.py) / CUDA-event time on the launching
    stream, summed over the timed region."""
    acc: dict = {}
    for name, s0, s1, nbytes in events:
        if name not in HBM_KERNELS:
            continue
        e = acc.setdefault(name, [0, 0.0, 0])
        e[0] += 1
        e[1] += s0.elapsed_time(s1)
        e[2] += nbytes
    out = {}
    for name, (n, ms, nb) in sorted(acc.items()):
        gbs = nb / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[name] = {"calls": n, "bytes": nb, "ms": ms, "gbs": gbs, "peak": peak_gbs,
                     "frac": gbs / peak_gbs if gbs else None}
    return out


def hbm_isolated(H: int, C: int, d: int, dev, peak_gbs: float, reps: int = 5) -> dict:
    """Each HBM-bound kernel of the path timed ALONE (CUDA events, `reps`
    back-to-back launches after a warm-up) on tensors of this rank's bench
    sizes: (H, C, d) bf16 activations, the fp32 transposed dQ accumulator,
    fp32 dK/dV-sized buffers. Complements the in-step `hbm_roofline`, whose
    kernels run at the power-capped clock of the attention step."""
    import torch

    from paper_2406_18485_b200 import kernels as K
    g = torch.Generator(device=dev).manual_seed(5)
    o = torch.randn((H, C, d), device=dev, generator=g).to(torch.bfloat16)
    do = torch.randn((H, C, d), device=dev, generator=g).to(torch.bfloat16)
    lse = torch.randn((H, C), device=dev, generator=g)
    acc = torch.randn((H, d, (C + 63) // 64 * 64), device=dev, generator=g)
    f32a = torch.randn((H, C, d), device=dev, generator=g)
    f32b = torch.randn((H, C, d), device=dev, generator=g)
    lse_b = torch.randn((H, C), device=dev, generator=g)
    idx = torch.arange(H, dtype=torch.int32, device=dev).flip(0)
    dst = torch.empty_like(o)
    a_hp = 4 if H % 4 == 0 else 1
    cases = {
        "a2d_bwd_preprocess": (lambda: K.bwd_preprocess(o, do, lse), H * C * (4 * d + 4) + H * ((C + 63) // 64 * 64) * 8),
        "a2d_dqt_to_bf16_d": (lambda: K.dqt_to_bf16(acc, C), H * C * d * 6),
        "a2d_gather_blocks": (lambda: K.gather_blocks(o, idx, dst), 2 * o.numel() * 2),
        "a2d_permute_blocks": (lambda: K.permute_blocks(o, a_hp, H // a_hp, out=dst), 2 * o.numel() * 2),
        "a2d_permute_f32_to_bf16": (lambda: K.permute_to_bf16(f32a, a_hp, H // a_hp, out=dst), 6 * f32a.numel()),
        "a2d_add_f32": (lambda: K.add_(f32a, f32b), 12 * f32a.numel()),
        "a2d_merge": (lambda: K.merge_(f32a, lse, f32b, lse_b), H * C * (12 * d + 12)),
    }
    out = {}
    for name, (fn, nbytes) in cases.items():
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"bytes": nbytes, "ms": ms, "gbs": gbs, "peak": peak_gbs, "frac": gbs / peak_gbs}
    del o, do, acc, f32a, f32b, dst
    torch.cuda.empty_cache()
    return out


def parity_check(a, run, op, q, k, v, do, world, rank):
    """Sampled f64-oracle parity of one step of the benched configuration on
    the benched inputs (oracle/sampled.py; checker only, outside every timed
    region). Gathers the SeqSharded tensors of all ranks to global order."""
    import torch
    import torch.distributed as dist

    from paper_2406_18485_b200.dist import unshard_global

    out = run.forward(q, k, v)
    dq, dk, dv = run.backward(do)
    lse = op.saved[3].contiguous() if run is op and op.saved is not None else None
    torch.cuda.synchronize()

    def glob(x):
        if world == 1:
            return unshard_global([x], op)
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x.contiguous())
        return unshard_global(parts, op)

    G = [glob(x) for x in (q, k, v, do, out, dq, dk, dv)]
    LSE = None
    if lse is not None:
        parts = [lse] if world == 1 else [torch.empty_like(lse) for _ in range(world)]
        if world > 1:
            dist.all_gather(parts, lse)
        LSE = torch.empty((a.heads, a.seq), dtype=torch.float32, device=lse.device)
        for r, part in enumerate(parts):
            hp, cp = op.grid.coords_of(r)
            LSE[hp * op.Hl:(hp + 1) * op.Hl][:, op.plans[cp].pos.long()] = part
    res = None
    if rank == 0:
        from oracle import sampled
        t0 = time.perf_counter()
        res = sampled.check(*G, LSE, causal=True, n_rows=512, n_keys=256, seed=7)
        res["violations"] = sampled.passes(res)
        res["seconds"] = time.perf_counter() - t0
        res["bar"] = ("per tensor [max_abs, rel_l2, max|ref|, excess]: rel-L2 <= 1e-2 and max-abs <= 2e-2 beyond "
                      "one bf16 ulp of |ref| for bf16 outputs (= the plain absolute bar where |ref| < ~5); "
                      "f64 row stats pinned <= 1e-9")
        res["sample"] = (f"{res['rows']} query rows x heads {res['heads']} (O, LSE, dQ), {res['keys']} keys "
                         f"(dK, dV) of this run's inputs, f64 oracle")
    del G
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--runtime", default="python", choices=["python", "native"],
                    help="python: dist.Attn2D (default); native: the C++ runtime behind a2d_ctx_create/a2d_fwd/a2d_bwd")
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--d-hp", type=int, default=0)
    ap.add_argument("--d-cp", type=int, default=0)
    ap.add_argument("--w", type=int, default=0)
    ap.add_argument("--placement", default="head_first")
    ap.add_argument("--cpu-rows", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", dest="check", action="store_true", default=True,
                    help="(default) after timing, check this run's O/LSE/dQ on sampled rows and dK/dV on sampled "
                         "keys against the f64 oracle (oracle/sampled.py) and report them under 'parity'")
    ap.add_argument("--no-check", dest="check", action="store_false")
    a = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world} (launch N>1 with torchrun)")

    import torch
    import torch.distributed as dist

    from paper_2406_18485_b200 import _lib
    from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig, Placement
    from paper_2406_18485_b200.dist import Attn2D

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29551")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    d_hp, d_cp, w = grid_of(a, world)
    S, H, Hkv, d = a.seq, a.heads, a.kv_heads, a.dim
    model = ModelConfig(seq_len=S, heads=H, kv_heads=Hkv, hidden=H * d)
    par = ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=w, placement=Placement(a.placement))
    op = Attn2D(model, par, ClusterConfig(), causal=True)
    if a.runtime == "native":
        from paper_2406_18485_b200.native import NativeAttn2D
        run = NativeAttn2D(model, par, ClusterConfig(), causal=True)
    else:
        run = op
    L = op.L
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q = torch.randn((H, L, d), device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn((Hkv, L, d), device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn((Hkv, L, d), device=dev, dtype=torch.bfloat16, generator=g)
    do = torch.randn((H, L, d), device=dev, dtype=torch.bfloat16, generator=g)

    def step():
        run.forward(q, k, v)
        return run.backward(do)

    for _ in range(max(a.warmup, 3 if a.warmup >= 3 else a.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()

    # ---------------- timed region: inputs resident in HBM
    clocks = ClockSampler(local)
    clocks.start()
    _lib.LOG.reset(timed=("a2d_fa_bwd_chunk", "a2d_fa_fwd_chunk") + HBM_KERNELS)
    _lib.LOG.enabled = True
    n_launch0 = _lib.launch_count()
    if a.runtime == "native":
        run.kernel_timing(True)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    _lib.LOG.enabled = False
    launches = _lib.launch_count() - n_launch0  # our kernels launched in the timed region (C-side counter)
    dist.barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    kern = {"a2d_fa_bwd_chunk": [0.0, 0], "a2d_fa_fwd_chunk": [0.0, 0]}
    for name, s0, s1, _ in _lib.LOG.events:
        if name in kern:
            kern[name][0] += s0.elapsed_time(s1)
            kern[name][1] += 1
    if a.runtime == "native":  # the C++ runtime brackets its own kernel launches
        km = run.kernel_ms()
        run.kernel_timing(False)
        kern = {"a2d_fa_bwd_chunk": [km["bwd_ms"], km["n_bwd"]], "a2d_fa_fwd_chunk": [km["fwd_ms"], km["n_fwd"]]}
    hbm = hbm_roofline(_lib.LOG.events, peaks()["hbm_gbs"])
    tt = torch.tensor([t_ms, kern["a2d_fa_bwd_chunk"][0], kern["a2d_fa_fwd_chunk"][0]], device=dev,
                      dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms, bwd_ms, fwd_ms = (float(x) for x in tt.tolist())

    flops = op.flops()
    value = flops * a.steps / (t_ms * 1e-3) / 1e12
    ms_step = t_ms / a.steps

    # ---------------- exposed communication: same step with every NCCL call
    # skipped (kernels and buffers identical), max over ranks
    exposed = None
    if world > 1:
        run.comm_enabled = False
        step()
        torch.cuda.synchronize()
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(a.steps):
            step()
        c1.record()
        torch.cuda.synchronize()
        run.comm_enabled = True
        tc = torch.tensor([c0.elapsed_time(c1)], device=dev, dtype=torch.float64)
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        t_comp = float(tc.item()) / a.steps
        exposed = {"ms_per_step": ms_step, "compute_only_ms_per_step": t_comp,
                   "exposed_ms": ms_step - t_comp, "frac": (ms_step - t_comp) / ms_step,
                   "definition": "t_layer - t_layer(comm disabled, same kernels), max over ranks"}
        dist.barrier()

    # ---------------- e2e through the same public API with host buffers.
    # Every step copies its q, k, v, dO from pinned host memory and its dq,
    # dk, dv back, inside the timed region; a side copy stream prefetches step
    # i+1's inputs and drains step i's gradients while compute runs (the usual
    # data-loader / offload pipelining; the first H2D and the last D2H are
    # exposed).
    e2e = None
    if not a.no_e2e:
        host_in = [x.cpu().pin_memory() for x in (q, k, v, do)]
        host_out = [[torch.empty((H, L, d), dtype=torch.bfloat16).pin_memory(),
                     torch.empty((Hkv, L, d), dtype=torch.bfloat16).pin_memory(),
                     torch.empty((Hkv, L, d), dtype=torch.bfloat16).pin_memory()] for _ in range(2)]
        dev_in = [[torch.empty_like(x, device=dev) for x in host_in] for _ in range(2)]
        h2d = sum(x.numel() * x.element_size() for x in host_in)
        d2h = sum(x.numel() * x.element_size() for x in host_out[0])
        cs = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream()

        def run_e2e(n):
            # per buffer set: one event when q/k/v landed (the forward waits for
            # it) and one when dO landed (only the backward waits for that)
            ev_qkv = [torch.cuda.Event() for _ in range(2)]
            ev_do = [torch.cuda.Event() for _ in range(2)]
            ev_done = [None, None]

            def load(j):
                for dst, src in zip(dev_in[j][:3], host_in[:3]):
                    dst.copy_(src, non_blocking=True)
                ev_qkv[j].record(cs)
                dev_in[j][3].copy_(host_in[3], non_blocking=True)
                ev_do[j].record(cs)

            with torch.cuda.stream(cs):
                cs.wait_stream(main)
                load(0)
            last = None
            for i in range(n):
                cur, nxt = i % 2, (i + 1) % 2
                main.wait_event(ev_qkv[cur])
                if i + 1 < n:
                    with torch.cuda.stream(cs):
                        if ev_done[nxt] is not None:
                            cs.wait_event(ev_done[nxt])  # step i-1 finished reading that buffer set
                        load(nxt)
                run.forward(dev_in[cur][0], dev_in[cur][1], dev_in[cur][2])
                main.wait_event(ev_do[cur])
                grads = run.backward(dev_in[cur][3])
                ev = torch.cuda.Event()
                ev.record(main)
                ev_done[cur] = ev
                with torch.cuda.stream(cs):
                    cs.wait_event(ev)
                    for dst, src in zip(host_out[cur], grads):
                        src.record_stream(cs)
                        dst.copy_(src, non_blocking=True)
                    last = torch.cuda.Event()
                    last.record(cs)
            main.wait_event(last)

        run_e2e(1)
        torch.cuda.synchronize()
        dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        run_e2e(a.steps)
        f1.record()
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], device=dev, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": flops * a.steps / (float(te.item()) * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "ms_per_step": float(te.item()) / a.steps,
               "pipelining": "side copy stream: H2D of step i+1 and D2H of step i overlap step i+1 compute; "
                              "dO's H2D overlaps the forward of its own step"}

    hbm_iso = None
    if rank == 0:
        try:
            hbm_iso = hbm_isolated(op.Hl, op.C, op.kd, dev, peaks()["hbm_gbs"])
        except Exception as exc:
            hbm_iso = {"error": f"{type(exc).__name__}: {exc}"}
    parity = None
    if a.check:
        try:
            parity = parity_check(a, run, op, q, k, v, do, world, rank)
        except Exception as exc:  # report, never lose the bench line
            parity = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        pk = peaks()
        per_gpu = value / world
        # dominant kernel: the backward chunk kernel (algorithmic FLOPs of the
        # backward = 2.5/3.5 of the step, split evenly over ranks)
        bwd_launch_flops = flops * (2.5 / 3.5) / world
        fwd_launch_flops = flops * (1.0 / 3.5) / world
        bwd_achieved = bwd_launch_flops * a.steps / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else None
        fwd_achieved = fwd_launch_flops * a.steps / (fwd_ms * 1e-3) / 1e12 if fwd_ms > 0 else None
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tr = json.load(f).get(f"bwd_S{S}_H{H}_d{d}_{d_hp}x{d_cp}")
                traffic = tr
        except (OSError, ValueError):
            pass
        roof = {"kernel": "a2d_fa_bwd_chunk (fa_bwd_q128_kernel, CTA pairs)", "bound": "tensor",
                "achieved": bwd_achieved, "peak": pk["bf16_tflops_sustained"], "unit": UNIT,
                "frac": (bwd_achieved / pk["bf16_tflops_sustained"]) if bwd_achieved else None,
                "frac_of_burst": (bwd_achieved / pk["bf16_tflops"]) if bwd_achieved else None,
                "peak_kind": f"{pk['src']} sustained (kernel runs inside a long step); burst {pk['bf16_tflops']}",
                "traffic": traffic,
                "share_of_step": bwd_ms / t_ms if t_ms else None,
                "fwd_kernel": {"achieved": fwd_achieved, "share_of_step": fwd_ms / t_ms if t_ms else None}}
        cpu = None
        if world == 1 and not a.no_cpu:
            with all_blas_threads():
                dt, fl = cpu_sample(a.cpu_rows, S, d)
                cores = cpu_cores()
            cpu = {"value": fl / dt / 1e12, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"1 head x last {a.cpu_rows} query rows x {S} keys, d={d}, causal fwd+bwd, "
                             f"f64 numpy oracle port, {dt:.2f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random bf16 q/k/v/dO)",
            "config": {**workload_config(a, world), **({"runtime": "native C++ (a2d_ctx_create/a2d_fwd/a2d_bwd)"}
                                                         if a.runtime == "native" else {})},
            "tflops_per_gpu": per_gpu, "mfu": per_gpu / pk["bf16_tflops"],
            "mfu_sustained": per_gpu / pk["bf16_tflops_sustained"],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "gpu_launches_per_step": launches / a.steps,
            "clocks": clk, "exposed_comm": exposed, "hbm_roofline": hbm,
            "hbm_roofline_isolated": hbm_iso, "parity": parity,
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
