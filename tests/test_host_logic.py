"""CPU tests of the host side: config/validation, layout index maps, ring
schedule + hop patterns (incl. the backward dK/dV route), the C ABI export
table, and the NCCL-free (gloo, world_size 2) exchange pattern."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import attn2d_oracle as orc
from paper_2406_18485_b200 import config as C
from paper_2406_18485_b200 import layout as Lo
from paper_2406_18485_b200 import schedule as Sc

REF_SRC = os.environ.get("ATTN2D_REF", "/root/reference/pkg/src")


# ------------------------------------------------------------------ config
def test_validate_messages_match_reference_kinds():
    m = C.ModelConfig(seq_len=48, heads=12, kv_heads=5, hidden=100)
    rep = C.validate(m, C.ParallelConfig(d_hp=5, d_cp=3, inner_ring=2), C.ClusterConfig())
    assert not rep.ok
    assert "H mod H_kv = 0" in rep.violations
    assert "D mod H = 0" in rep.violations
    assert "d_hp divides H" in rep.violations
    assert "w divides d_cp" in rep.violations
    assert "S mod (2 * d_sp) = 0" in rep.violations
    ok = C.validate(C.ModelConfig(seq_len=64, heads=8, kv_heads=2, hidden=64),
                    C.ParallelConfig(d_hp=2, d_cp=4, inner_ring=2), C.ClusterConfig())
    assert ok.ok
    with pytest.raises(ValueError):
        C.check_config(m, C.ParallelConfig(d_hp=5, d_cp=3), C.ClusterConfig())


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_validate_identical_to_reference():
    import sys
    sys.path.insert(0, REF_SRC)
    import attn2d
    rng = np.random.default_rng(0)
    for _ in range(300):
        s, h, hk, hid = (int(x) for x in rng.integers(1, 40, 4))
        dh, dc, w = (int(x) for x in rng.integers(0, 9, 3))
        pl = [C.Placement.HEAD_FIRST, C.Placement.CONTEXT_FIRST][int(rng.integers(2))]

        def run(mod, M, P, Cl, Pl):
            try:
                return mod(M(s, h, hk, hid), P(dh, dc, inner_ring=w, placement=Pl), Cl()).violations
            except ZeroDivisionError:
                return "ZeroDivisionError"

        ours = run(C.validate, C.ModelConfig, C.ParallelConfig, C.ClusterConfig, pl)
        ref = run(attn2d.validate, attn2d.ModelConfig, attn2d.ParallelConfig, attn2d.ClusterConfig,
                  attn2d.Placement(pl.value))
        assert ours == ref


@pytest.mark.parametrize("placement", list(C.Placement))
def test_rank_grid_bijection(placement):
    g = C.RankGrid(4, 2, placement, 8)
    seen = set()
    for r in range(8):
        hp, cp = g.coords_of(r)
        assert g.rank_of(hp, cp) == r
        seen.add((hp, cp))
    assert len(seen) == 8
    if placement is C.Placement.HEAD_FIRST:
        assert g.hp_group(1) == [4, 5, 6, 7]
    else:
        assert g.cp_group(1) == [2, 3]


def test_replicated_heads():
    assert C.replicated_kv_heads(8, 4, 32) == 8
    assert C.replicated_kv_heads(8, 16, 32) == 16
    # reference quirk: validate accepts H=12, H_kv=6, d_hp=4 but the
    # replicated head count stays 6, which the scatter then rejects
    assert C.replicated_kv_heads(6, 4, 12) == 6
    with pytest.raises(ValueError):
        C.replicated_kv_heads(8, 64, 32)
    assert list(Lo.replica_source_heads(2, 4)) == [0, 0, 1, 1]


# ------------------------------------------------------------------ layout
def test_layout_matches_reference_golden():
    g = golden("layouts.npz")
    for s, d_cp in ((8, 1), (8, 2), (48, 4), (64, 8), (4096, 2), (128, 4)):
        perm, inv = Lo.zigzag_reorder(s, d_cp)
        assert np.array_equal(perm, g[f"zz_{s}_{d_cp}_perm"])
        assert np.array_equal(inv, g[f"zz_{s}_{d_cp}_inv"])
    for d_hp, d_cp in ((1, 1), (2, 2), (4, 2), (2, 4), (1, 8), (8, 1)):
        for pl in C.Placement:
            grid = C.RankGrid(d_hp, d_cp, pl, 8)
            tag = f"{d_hp}x{d_cp}_{pl.value}"
            seq = np.stack([Lo.seq_positions(64, grid, *grid.coords_of(r)) for r in range(grid.d_sp)])
            head = np.stack([Lo.cp_positions(64, d_cp, grid.coords_of(r)[1]) for r in range(grid.d_sp)])
            assert np.array_equal(seq, g[f"seqpos_{tag}"])
            assert np.array_equal(head, g[f"headpos_{tag}"])


def test_stripe_bases_describe_cp_chunk():
    for s, d_cp in ((64, 4), (4096, 2)):
        for j in range(d_cp):
            b0, b1, sig = Lo.stripe_bases(s, d_cp, j)
            want = np.concatenate([np.arange(b0, b0 + sig), np.arange(b1, b1 + sig)])
            assert np.array_equal(Lo.cp_positions(s, d_cp, j), want)


def test_zigzag_balance():
    for d_cp in (2, 4, 8):
        counts = [int((Lo.cp_positions(32 * d_cp, d_cp, j) + 1).sum()) for j in range(d_cp)]
        assert len(set(counts)) == 1


# ------------------------------------------------------------------ schedule
@pytest.mark.parametrize("d_cp", [1, 2, 3, 4, 6, 8])
def test_schedules_walks_and_dkv_routes(d_cp):
    for w in (x for x in range(1, d_cp + 1) if d_cp % x == 0):
        sch = Sc.build_ring_schedule(d_cp, w)
        assert [[s.source for s in row] for row in sch.steps] == orc.ring_sources(d_cp, w)
        Sc.check_walk(sch)
        Sc.check_dkv_route(sch)


def test_schedule_kats():
    assert [s.source for s in Sc.build_ring_schedule(8, 4).steps[0]] == [0, 3, 2, 1, 4, 7, 6, 5]
    assert [s.source for s in Sc.build_ring_schedule(4, 2).steps[1]] == [1, 0, 3, 2]
    with pytest.raises(ValueError):
        Sc.build_ring_schedule(8, 3)


# ------------------------------------------------------------------ C ABI
def _header_symbols():
    text = open(os.path.join(ROOT, "include", "attn2d_sm100.h")).read()
    return sorted(set(re.findall(r"\b(a2d_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2406_18485_b200 import _lib
    from paper_2406_18485_b200 import build as B
    B.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/attn2d_sm100.h but not exported"
    loaded = _lib.load()
    assert loaded.a2d_abi_version() == 2
    assert set(_lib.SIGNATURES) | {"a2d_last_error", "a2d_abi_version", "a2d_launch_count"} == set(syms)
    assert _lib.launch_count() == 0  # nothing launched without a GPU


def test_library_rejects_bad_shapes_without_gpu():
    """Argument validation happens before any CUDA call (ValueError analogue)."""
    from paper_2406_18485_b200 import _lib
    with pytest.raises(ValueError, match="head dim"):
        _lib.call("a2d_fa_fwd_chunk", None, None, None, None, None, None, None, 4, 2, 16, 16, 96, 1, 0.1, 0,
                  None, None, None, None)
    with pytest.raises(ValueError, match="not divisible"):
        _lib.call("a2d_fa_fwd_chunk", None, None, None, None, None, None, None, 6, 4, 16, 16, 128, 1, 0.1, 0,
                  None, None, None, None)
    with pytest.raises(ValueError, match="% 16"):
        _lib.call("a2d_permute_blocks", None, None, 2, 2, 24, None)


# ------------------------------------------------------------------ gloo exchange
def _gloo_worker(rank, world, port, d_cp, w, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sch = Sc.build_ring_schedule(d_cp, w)
        pe = Sc.ring_peers(rank, d_cp, w)
        cur = torch.tensor([rank])
        first = cur.clone()
        got = [int(cur)]
        for s, step in enumerate(sch.steps[rank]):
            if s == d_cp - 1:
                break
            nxt = torch.empty(1, dtype=torch.long)
            if (s + 1) % w:
                send, to, frm = cur, pe.inner_to, pe.inner_from
            else:
                send, to, frm = first, pe.outer_to, pe.outer_from
            ops = [dist.P2POp(dist.isend, send, to), dist.P2POp(dist.irecv, nxt, frm)]
            for wk in dist.batch_isend_irecv(ops):
                wk.wait()
            cur = nxt
            if (s + 1) % w == 0:
                first = cur.clone()
            got.append(int(cur))
        # dK/dV accumulator route: (chunk id, number of ranks that added to it)
        acc = torch.tensor([sch.steps[rank][0].source, 1])
        ok = True
        for s in range(d_cp):
            kind = Sc.dkv_hop(s, d_cp, w)
            to, frm = (pe.inner_to, pe.inner_from) if kind == "inner" else (pe.diag_to, pe.diag_from)
            nxt = torch.empty_like(acc)
            for wk in dist.batch_isend_irecv([dist.P2POp(dist.isend, acc, to), dist.P2POp(dist.irecv, nxt, frm)]):
                wk.wait()
            acc = nxt
            if s + 1 < d_cp:
                ok &= int(acc[0]) == sch.steps[rank][s + 1].source
                acc[1] += 1
        q.put((rank, got, [s.source for s in sch.steps[rank]], [int(acc[0]), int(acc[1]), ok]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d_cp,w", [(2, 1), (2, 2)])
def test_gloo_ring_exchange(d_cp, w):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + d_cp * 10 + w
    ps = [ctx.Process(target=_gloo_worker, args=(r, d_cp, port, d_cp, w, q)) for r in range(d_cp)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, got, want, acc in res:
        assert got == want, (rank, got, want)
        assert acc == [rank, d_cp, True], (rank, acc)  # home, visited by every CP rank, in order


@pytest.mark.parametrize("d_hp,Hl,Hkl,ng", [(2, 16, 16, 1), (4, 8, 2, 1), (2, 16, 16, 4), (8, 4, 4, 2), (2, 4, 1, 1)])
def test_symm_exchange_layout_fits_and_is_disjoint(d_hp, Hl, Hkl, ng):
    """Byte layout of the symmetric-memory exchange buffer (dist.Attn2D._xoff):
    every exchange fits inside the allocation, and exchanges that can be in
    flight together (all groups of one phase; q with kv; dq with dk and dv;
    the fp32 GQA gathers) never overlap."""
    from types import SimpleNamespace
    from paper_2406_18485_b200.dist import Attn2D
    L, bd = 1024, 128
    op = SimpleNamespace(par=SimpleNamespace(d_hp=d_hp), L=L, bd=bd, Hl=Hl, Hkl=Hkl, ng=ng,
                         Hq_g=Hl // ng, Hk_g=Hkl // ng)
    tok = L * bd
    op._in_bytes = d_hp * tok * 2 * (Hl + 2 * Hkl)
    total = op._in_bytes + d_hp * tok * (2 * Hl + 4 * 2 * Hkl)
    off = lambda name, g=0: Attn2D._xoff(op, name, g)  # noqa: E731
    q_b, kv_b, k_b = d_hp * tok * 2 * op.Hq_g, d_hp * tok * 2 * 2 * op.Hk_g, d_hp * tok * 2 * op.Hk_g
    phases = [
        [(off("q", g), q_b) for g in range(ng)] + [(off("kv", g), kv_b) for g in range(ng)],   # fwd in
        [(off("do", g), q_b) for g in range(ng)],                                              # bwd in
        [(off("out", g), q_b) for g in range(ng)],                                             # fwd out
        [(off(n, g), b) for g in range(ng) for n, b in (("dq", q_b), ("dk", k_b), ("dv", k_b))],  # bwd out
    ]
    if ng == 1:
        phases.append([(off("dq"), q_b), (off("dk32"), 2 * k_b), (off("dv32"), 2 * k_b)])  # GQA replicas
    for spans in phases:
        for o, b in spans:
            assert 0 <= o and o + b <= total
        spans = sorted(spans)
        for (o1, b1), (o2, _) in zip(spans, spans[1:]):
            assert o1 + b1 <= o2, spans
    # scatters use the IN region, gathers the OUT region
    assert all(o + b <= op._in_bytes for o, b in phases[0] + phases[1])
    assert all(o >= op._in_bytes for o, _ in phases[2] + phases[3])


@pytest.mark.parametrize("d_cp,w", [(1, 1), (2, 1), (2, 2), (4, 1), (4, 2), (4, 4), (8, 2), (8, 4), (16, 4), (12, 3)])
def test_native_ring_plan_matches_schedule(d_cp, w):
    """The native runtime's C++ ring plan (a2d_ring_plan) equals schedule.py's
    schedule and peers, and its zig-zag positions equal layout.cp_positions."""
    import ctypes
    import numpy as np
    from paper_2406_18485_b200 import _lib
    from paper_2406_18485_b200.layout import cp_positions
    from paper_2406_18485_b200.schedule import build_ring_schedule, ring_peers
    sched = build_ring_schedule(d_cp, w)
    S = 48 * d_cp
    for j in range(d_cp):
        steps = (ctypes.c_int32 * (3 * d_cp))()
        peers = (ctypes.c_int32 * 6)()
        _lib.call("a2d_ring_plan", d_cp, w, j, ctypes.addressof(steps), ctypes.addressof(peers))
        want = [(st.source, st.outer, st.inner) for st in sched.steps[j]]
        got = [tuple(steps[3 * i:3 * i + 3]) for i in range(d_cp)]
        assert got == want, (j, got, want)
        p = ring_peers(j, d_cp, w)
        assert list(peers) == [p.inner_to, p.inner_from, p.outer_to, p.outer_from, p.diag_to, p.diag_from]
        pos = np.zeros(S // d_cp, dtype=np.int32)
        _lib.call("a2d_zigzag_positions", S, d_cp, j, pos.ctypes.data)
        assert np.array_equal(pos, cp_positions(S, d_cp, j))
    with pytest.raises(ValueError):
        _lib.call("a2d_ring_plan", d_cp, d_cp + 1, 0, ctypes.addressof(steps), ctypes.addressof(peers))


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the driver's reference arm) prints one JSON
    line with the contract's fields, on the same config object as our arm."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--seq", "4096", "--cpu-rows", "64"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["config"]["workload"].startswith("2D-Attention fwd+bwd") and line["config"]["global_tokens"] == 4096


# ------------------------------------------------------------------ data-parallel replicas
def _replica_worker(rank, world, port, d_hp, d_cp, interleave, q):
    import torch
    import torch.distributed as dist

    from paper_2406_18485_b200.config import ClusterConfig, ParallelConfig, build_rank_grid
    from paper_2406_18485_b200.dist import make_groups
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_rep = world // (d_hp * d_cp)
        reps = [list(range(r, world, n_rep)) if interleave else list(range(r * d_hp * d_cp, (r + 1) * d_hp * d_cp))
                for r in range(n_rep)]
        # each replica group created by all ranks (torch's rule), in the same order
        pgs = [dist.new_group(r) for r in reps]
        mine = next(i for i, r in enumerate(reps) if rank in r)
        grid = build_rank_grid(ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=1), ClusterConfig())
        hp_group, ring, g_ranks = make_groups(grid, pgs[mine])
        out = {"rank": rank, "replica": reps[mine], "g": g_ranks}
        if hp_group is not None:
            out["hp"] = sorted(dist.get_process_group_ranks(hp_group))
            t = torch.tensor([rank])
            dist.all_reduce(t, group=hp_group)  # traffic stays inside this replica's HP group
            out["hp_sum"] = int(t)
        if ring[0] is not None:
            out["ring"] = [sorted(dist.get_process_group_ranks(g)) for g in ring]
            t = torch.tensor([rank])
            dist.all_reduce(t, group=ring[1])
            out["ring_sum"] = int(t)
        q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d_hp,d_cp,interleave", [(1, 2, False), (2, 1, True), (1, 2, True)])
def test_make_groups_for_data_parallel_replicas(d_hp, d_cp, interleave):
    """Two data-parallel replicas (d_dp = 2): every rank creates the HP
    and ring groups of both replicas in one global order, so the groups are
    consistent (no cross-wired or hanging communicators) and stay inside the
    replica."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2 * d_hp * d_cp
    port = 29650 + 10 * d_hp + d_cp + (5 if interleave else 0)
    ps = [ctx.Process(target=_replica_worker, args=(r, world, port, d_hp, d_cp, interleave, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for r in res:
        assert r["g"] == r["replica"]
        if "hp" in r:
            assert set(r["hp"]) <= set(r["replica"]) and len(r["hp"]) == d_hp
            assert r["hp_sum"] == sum(r["hp"])
        if "ring" in r:
            assert all(set(g) <= set(r["replica"]) and len(g) == d_cp for g in r["ring"])
            assert r["ring_sum"] == sum(r["ring"][1])
