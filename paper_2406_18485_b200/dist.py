"""SPMD 2D-Attention runtime: one process per GPU over NVLink.

Alg. 1 of the paper (ref ``ring.py:82-119``) executed for real:

  SeqSharded q/k/v (H, L, d) per rank (head-major, or token-major views of a
  fused QKV projection)
    -> pack (128-bit gather kernel; GQA replication by addressing)
    -> all-to-all inside the HP group (d_hp ranks sharing a cp_index): by
       default copy-engine writes straight into the peers' torch
       symmetric-memory buffers + a device barrier (``_xchg``); NCCL
       ``all_to_all_single`` with A2D_TRANSPORT=nccl
    -> unpack (128-bit permute kernel) = HeadSharded (H/d_hp, C, d)
    -> Double-Ring attention inside the CP group (d_cp ranks sharing an
       hp_index): KV chunks rotate over an inner ring of size w and an outer
       ring of d_cp/w, as NCCL send/recv on separate communicators so an
       outer hop (issued at the start of an outer step) overlaps the w inner
       hops and the attention kernels (Alg. 2);
       each step folds its block into an fp32 accumulator inside the
       attention kernel's epilogue
    -> pack + all-to-all back -> SeqSharded output (H, L, d)

Backward (not in the reference; designed here and checked
against the global oracle): KV chunks rotate again along the same schedule;
a travelling fp32 dK/dV accumulator follows each chunk one step behind and
is added to (K4 kernel) by every rank that consumes the chunk. The
accumulator's hop is (r, p) -> (r, p+1) inside an outer step and the
"diagonal" (r, p) -> (r+1, p+1) across outer steps; the same diagonal hop
after the last step brings every accumulator home to its owner (in bf16
when nothing is added at home). dQ accumulates in a transposed fp32 buffer
that the gradient all-to-all's pack turns into bf16.

Communication never blocks the host: ``Work.wait()`` / stream events only
make the compute stream wait.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from .config import (ClusterConfig, ModelConfig, ParallelConfig, build_rank_grid,
                     check_config, replicated_kv_heads)
from .layout import cp_positions, replica_source_heads, seq_positions
from .schedule import build_ring_schedule, dkv_hop, ring_peers


@dataclass
class StepTimes:
    """CUDA events per phase of the last call (for bench / exposed-comm)."""

    events: list = field(default_factory=list)

    def mark(self, name: str):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.append((name, e))

    def clear(self):
        self.events.clear()


def make_groups(grid, group=None):
    """(hp_group, (ring_inner, ring_outer, ring_dkv), replica_ranks) of this rank.

    ``group`` (default WORLD) is this rank's replica: d_hp*d_cp ranks running
    one 2D-attention layer; several data-parallel replicas may run side by
    side. torch needs every WORLD rank to call new_group for every group, with
    the same ranks, in the same order — so the replicas' rank lists are
    gathered first and every rank creates the HP and ring groups of EVERY
    replica in one global order (sorted replicas, then HP groups by cp, then
    ring groups by hp)."""
    world = dist.get_world_size()
    if group is None:
        mine = list(range(world))
        replicas = [tuple(mine)]
    else:
        mine = dist.get_process_group_ranks(group)
        allr = [None] * world
        dist.all_gather_object(allr, list(mine))
        replicas = sorted({tuple(r) for r in allr})
        flat = sorted(r for rep in replicas for r in rep)
        if flat != list(range(world)) or any(len(rep) != grid.d_sp for rep in replicas):
            raise ValueError("replica groups must partition WORLD into groups of d_hp*d_cp ranks")
    me = dist.get_rank()
    hp_i, cp_j = grid.coords_of(mine.index(me))
    hp_group, ring = None, (None, None, None)
    for rep in replicas:
        own = list(rep) == list(mine)
        for j in range(grid.d_cp):
            g = dist.new_group([rep[r] for r in grid.hp_group(j)]) if grid.d_hp > 1 else None
            if own and j == cp_j:
                hp_group = g
        for i in range(grid.d_hp):
            ranks = [rep[r] for r in grid.cp_group(i)]
            gs = tuple(dist.new_group(ranks) if grid.d_cp > 1 else None for _ in range(3))
            if own and i == hp_i:
                ring = gs
    return hp_group, ring, list(mine)


class _State(tuple):
    """(qh, kvh, out_h, lse) of one forward. ``guard`` = (tensor, version) when
    qh aliases the caller's q (d_hp = 1, head-major bf16 input): the backward
    refuses to run if q was modified in place in between (it would silently
    produce wrong gradients otherwise)."""

    guard = None


class Attn2D:
    """Per-rank 2D-Attention operator (HP all-to-all x Double-Ring CP).

    ``forward(q, k, v)`` takes this rank's SeqSharded chunks
    (H, L, d) / (H_kv, L, d) in the zig-zag token order of
    ``layout.seq_positions`` and returns the SeqSharded output (H, L, d).
    ``backward(dout)`` returns (dq, dk, dv) in the same layout.
    """

    def __init__(self, model: ModelConfig, par: ParallelConfig, cluster: ClusterConfig | None = None,
                 causal: bool = True, group=None, device=None):
        cluster = cluster or ClusterConfig()
        check_config(model, par, cluster)
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised (one rank per GPU)")
        self.model, self.par, self.causal = model, par, causal
        self.grid = build_rank_grid(par, cluster)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != self.grid.d_sp:
            raise ValueError(f"world size {self.world} != d_hp*d_cp = {self.grid.d_sp}")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.hp, self.cp = self.grid.coords_of(self.rank)
        d_hp, d_cp, w = par.d_hp, par.d_cp, par.inner_ring
        S, H, Hkv = model.seq_len, model.heads, model.kv_heads
        self.d = model.head_dim
        self.kd = K.fwd_dim(self.d)
        self.bd = self.kd  # backward kernel head dim (64 or 128, zero-padded like the forward)
        self.scale = 1.0 / math.sqrt(self.d)
        self.H_rep = replicated_kv_heads(Hkv, d_hp, H)
        if self.H_rep % d_hp != 0:
            raise ValueError(f"{self.H_rep} heads not divisible by d_hp={d_hp}")
        self.Hl, self.Hkl = H // d_hp, self.H_rep // d_hp
        self.rep = self.H_rep // Hkv
        self.L, self.C = S // self.grid.d_sp, S // d_cp
        self.C_pad = (self.C + 63) // 64 * 64

        # ---- process groups (created by every rank, in the same order)
        self.hp_group, (self.ring_inner, self.ring_outer, self.ring_dkv), self._g = make_groups(self.grid, group)

        # ---- schedule and peers (global ranks)
        self.schedule = build_ring_schedule(d_cp, w)
        self.steps = self.schedule.steps[self.cp]
        pe = ring_peers(self.cp, d_cp, w)

        def cp_rank(j):
            return self._g[self.grid.rank_of(self.hp, j)]

        self.inner_to, self.inner_from = cp_rank(pe.inner_to), cp_rank(pe.inner_from)
        self.outer_to, self.outer_from = cp_rank(pe.outer_to), cp_rank(pe.outer_from)
        self.diag_to, self.diag_from = cp_rank(pe.diag_to), cp_rank(pe.diag_from)

        # ---- positions / tile plans (device)
        dev = self.device
        self.seq_pos = seq_positions(S, self.grid, self.hp, self.cp)
        self.plans = [K.ChunkPlan(torch.as_tensor(cp_positions(S, d_cp, j), dtype=torch.int32, device=dev))
                      for j in range(d_cp)]
        # pack maps for the KV all-to-all: destination block (peer, t, hl) of
        # [d_hp][2][Hkl] reads original head src(peer*Hkl + hl) of k (t=0) or v (t=1)
        src = replica_source_heads(Hkv, self.H_rep)
        dmap_k, dmap_v, smap = [], [], []
        for peer in range(d_hp):
            for hl in range(self.Hkl):
                smap.append(int(src[peer * self.Hkl + hl]))
                dmap_k.append(peer * 2 * self.Hkl + hl)
                dmap_v.append(peer * 2 * self.Hkl + self.Hkl + hl)
        self._smap = torch.tensor(smap, dtype=torch.int32, device=dev)
        self._dmap_k = torch.tensor(dmap_k, dtype=torch.int32, device=dev)
        self._dmap_v = torch.tensor(dmap_v, dtype=torch.int32, device=dev)
        # ---- head groups: the HP exchange of group g+1 (and the output gather
        # of group g) run on NCCL's stream while group g's ring attention runs
        self.ng = self._choose_groups()
        self.Hq_g, self.Hk_g = self.Hl // self.ng, self.Hkl // self.ng
        if self.ng > 1:
            it = lambda xs: torch.tensor(xs, dtype=torch.int32, device=dev)  # noqa: E731
            self._qmap, self._kmap, self._kvsrc, self._kvdk, self._kvdv = [], [], [], [], []
            for g in range(self.ng):
                self._qmap.append(it([p * self.Hl + g * self.Hq_g + j for p in range(d_hp) for j in range(self.Hq_g)]))
                self._kmap.append(it([p * self.Hkl + g * self.Hk_g + j for p in range(d_hp) for j in range(self.Hk_g)]))
                self._kvsrc.append(it([int(src[p * self.Hkl + g * self.Hk_g + j])
                                       for p in range(d_hp) for j in range(self.Hk_g)]))
                self._kvdk.append(it([p * 2 * self.Hk_g + j for p in range(d_hp) for j in range(self.Hk_g)]))
                self._kvdv.append(it([p * 2 * self.Hk_g + self.Hk_g + j for p in range(d_hp) for j in range(self.Hk_g)]))
            self._iota = it(list(range(d_hp * max(self.Hq_g, self.Hk_g))))
        self._bufs: dict = {}
        # ---- HP exchange transport: "symm" = copy-engine writes into the peers'
        # symmetric-memory buffers + a device barrier (no SMs taken, ~770 GB/s
        # per direction); "nccl" = all_to_all_single. A2D_TRANSPORT overrides.
        self.transport = "nccl"
        self._symm = None
        if d_hp > 1 and os.environ.get("A2D_TRANSPORT", "symm") == "symm":
            self._init_symm()
        self.times = StepTimes()
        self.record_times = False
        self.saved = None
        # False = "compute only": identical kernels and buffers, every NCCL call
        # skipped (receive buffers keep pre-staged data). Only for measuring
        # exposed communication (t_layer - t_compute_only, ref timeline.py:152).
        self.comm_enabled = True

    def _init_symm(self) -> None:
        """Symmetric buffer of this HP group: IN region (scatters: q + kv, or
        dO) and OUT region (gathers: O, or dQ + dK + dV, fp32 when GQA replicas
        are summed after the gather). Collective over the HP group."""
        try:
            import torch.distributed._symmetric_memory as symm
        except ImportError:
            return
        d_hp, tok = self.par.d_hp, self.L * self.bd
        self._in_bytes = d_hp * tok * 2 * (self.Hl + 2 * self.Hkl)
        out_bytes = d_hp * tok * (2 * self.Hl + 4 * 2 * self.Hkl)
        ok = True
        try:  # e.g. an HP group spanning nodes cannot map peer memory: keep NCCL
            buf = symm.empty(self._in_bytes + out_bytes, dtype=torch.uint8, device=self.device)
            self._symm = symm.rendezvous(buf, self.hp_group.group_name)
        except Exception:  # noqa: BLE001 - any failure means "no symmetric memory here"
            ok = False
        # every HP rank must pick the same transport, or the group deadlocks
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=self.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.hp_group)
        if not ok or int(flag.item()) == 0:
            self._symm = None
            return
        self._symm_buf = buf
        self._peer = [self._symm.get_buffer(r, (buf.numel(),), torch.uint8) for r in range(d_hp)]
        self._xstreams = [torch.cuda.Stream(self.device) for _ in range(d_hp - 1)]
        self._xstream_bar = torch.cuda.Stream(self.device)
        self.transport = "symm"

    # byte offsets of each exchange inside the symmetric buffer (static layout:
    # a region is only rewritten after every peer passed a later barrier)
    def _xoff(self, name: str, g: int = 0) -> int:
        d_hp, tok = self.par.d_hp, self.L * self.bd
        q_bytes = d_hp * tok * 2 * self.Hq_g   # one head group of a query-like tensor
        kv_bytes = d_hp * tok * 2 * 2 * self.Hk_g
        k_bytes = d_hp * tok * 2 * self.Hk_g
        ng = self.ng
        if name in ("q", "do"):
            return g * q_bytes
        if name == "kv":
            return ng * q_bytes + g * kv_bytes
        base = self._in_bytes
        if name in ("out", "dq"):
            return base + g * q_bytes
        if name in ("dk", "dv"):
            return base + ng * q_bytes + (0 if name == "dk" else ng * k_bytes) + g * k_bytes
        if name in ("dk32", "dv32"):  # fp32, ng == 1
            return base + q_bytes + (0 if name == "dk32" else 2 * k_bytes)
        raise KeyError(name)

    def _xchg(self, send: torch.Tensor, name: str, g: int = 0, wait: bool = True):
        """All-to-all of send [d_hp][...] -> recv [d_hp][...] (recv[p] = peer p's
        send[me]). "symm": one copy-engine write per peer straight into its
        buffer, then a device barrier. Returns recv (and, wait=False, an event
        the consumer stream must wait for)."""
        if self.transport != "symm":
            recv = self._buf(f"{name}.recv{g}", send.shape, send.dtype)
            w = None
            if self.comm_enabled:
                w = dist.all_to_all_single(recv, send, group=self.hp_group, async_op=not wait)
            return recv if wait else (recv, w)
        d_hp, me = self.par.d_hp, self.hp
        nb = send[0].numel() * send.element_size()
        off = self._xoff(name, g)
        recv = self._symm_buf[off:off + d_hp * nb].view(send.dtype).view(send.shape)
        main = torch.cuda.current_stream()
        bar = self._xstream_bar
        src = send.view(torch.uint8).view(d_hp, nb)
        if self.comm_enabled:
            ev = torch.cuda.Event()
            ev.record(main)
            for i in range(d_hp - 1):
                p = (me + 1 + i) % d_hp
                s = self._xstreams[i]
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    self._peer[p][off + me * nb:off + (me + 1) * nb].copy_(src[p], non_blocking=True)
                bar.wait_stream(s)
        else:
            bar.wait_stream(main)
        with torch.cuda.stream(bar):
            bar.wait_stream(main)
            recv[me].copy_(send[me], non_blocking=True)
            if self.comm_enabled:
                self._symm.barrier()
        done = torch.cuda.Event()
        done.record(bar)
        if wait:
            main.wait_event(done)
            return recv
        return recv, done

    def _choose_groups(self) -> int:
        """Head groups for the pipelined exchange (1 = one exchange per phase).
        Opt-in via A2D_HEAD_GROUPS=g: measured on B200 the
        overlap loses — NCCL's all-to-all kernels take SMs from the attention
        kernels for longer than the transfer they hide (N=4: 3705 vs 3820
        TFLOP/s). Needs d_hp > 1, d = 128, no GQA replicas and even splits."""
        env = os.environ.get("A2D_HEAD_GROUPS")
        if not env or self.par.d_hp == 1 or self.d != self.bd or self.kd != self.bd or self.rep != 1:
            return 1
        g = int(env)
        return g if g >= 1 and self.Hl % g == 0 and self.Hkl % g == 0 else 1

    # ------------------------------------------------------------ helpers
    def _buf(self, name: str, shape, dtype) -> torch.Tensor:
        key = (name, tuple(shape), dtype)
        t = self._bufs.get(key)
        if t is None:
            t = torch.empty(shape, dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t

    def _mark(self, name):
        if self.record_times:
            self.times.mark(name)

    # ---- grouped exchange (ng > 1): packs / unpacks of head group g
    def _send_q_g(self, x: torch.Tensor, g: int, name: str, tm: bool) -> torch.Tensor:
        """[d_hp][Hq_g][L][d] bf16 send buffer of query-like tensor x for group g."""
        d_hp, dk = self.par.d_hp, self.bd
        send = self._buf(f"{name}.send{g}", (d_hp, self.Hq_g, self.L, dk), torch.bfloat16)
        if tm and x.dtype == torch.bfloat16 and x.stride(-1) == 1:
            K.copy_rows(x, send.view(d_hp * self.Hq_g, self.L, dk).transpose(0, 1), self._qmap[g])
        else:
            x = K.pad_dim(x.transpose(0, 1) if tm else x, dk)
            K.gather_blocks(x, self._qmap[g], send)
        return send

    def _send_kv_g(self, k: torch.Tensor, v: torch.Tensor, g: int, tm: bool) -> torch.Tensor:
        d_hp, dk = self.par.d_hp, self.bd
        send = self._buf(f"kv.send{g}", (d_hp, 2, self.Hk_g, self.L, dk), torch.bfloat16)
        if tm and k.dtype == v.dtype == torch.bfloat16 and k.stride(-1) == 1 and v.stride(-1) == 1:
            rows = send.view(d_hp * 2 * self.Hk_g, self.L, dk).transpose(0, 1)
            K.copy_rows(k, rows, self._kvsrc[g], self._kvdk[g])
            K.copy_rows(v, rows, self._kvsrc[g], self._kvdv[g])
        else:
            if tm:
                k, v = k.transpose(0, 1), v.transpose(0, 1)
            k, v = K.pad_dim(k, dk), K.pad_dim(v, dk)
            K.gather_blocks(k, self._kvsrc[g], send, self._kvdk[g])
            K.gather_blocks(v, self._kvsrc[g], send, self._kvdv[g])
        return send

    def _unpack_g(self, recv: torch.Tensor, hmap: torch.Tensor, out: torch.Tensor, tm: bool) -> None:
        """recv [d_hp][Hn][L][d] -> the caller's SeqSharded tensor at heads hmap."""
        n = recv.shape[0] * recv.shape[1]
        flat = recv.view(n, self.L, recv.shape[-1])
        if tm:
            K.copy_rows(flat.transpose(0, 1), out, None, hmap)
        else:
            K.gather_blocks(flat, self._iota[:n], out, hmap)

    def _new(self, name: str, shape, dtype, fresh: bool) -> torch.Tensor:
        """Workspace buffer, or newly allocated memory when the result outlives the call."""
        return torch.empty(shape, dtype=dtype, device=self.device) if fresh else self._buf(name, shape, dtype)

    def _head_major_send(self, x: torch.Tensor, name: str, dk: int, token_major: bool,
                         fresh: bool = False) -> torch.Tensor:
        """This rank's (H, L, dk) head-major bf16 send buffer for the HP all-to-all.

        Token-major (L, H, d) input — possibly a strided head slice of a fused
        QKV projection output — is converted by the pack itself (one pass)."""
        if token_major and x.shape[-1] == dk and x.dtype == torch.bfloat16 and x.stride(-1) == 1:
            send = self._new(name + ".send", (x.shape[1], self.L, dk), torch.bfloat16, fresh)
            K.copy_rows(x, send.transpose(0, 1))
            return send
        if token_major:
            x = x.transpose(0, 1)
        return K.pad_dim(x, dk)

    def _scatter_q(self, x: torch.Tensor, name: str, dk: int, token_major: bool = False,
                   fresh: bool = False) -> torch.Tensor:
        """SeqSharded (H, L, d) [or token-major (L, H, d)] -> HeadSharded (Hl, C, dk) bf16.
        fresh=True: the result owns its memory (it is kept for the backward)."""
        d_hp = self.par.d_hp
        x = self._head_major_send(x, name, dk, token_major, fresh and d_hp == 1)
        if d_hp == 1:
            return x
        recv = self._xchg(x.view(d_hp, self.Hl, self.L, dk), name)
        out = self._new(name, (self.Hl, self.C, dk), torch.bfloat16, fresh)
        return K.permute_blocks(recv, d_hp, self.Hl, out=out)

    def _scatter_kv(self, k: torch.Tensor, v: torch.Tensor, name: str, dk: int,
                    token_major: bool = False, fresh: bool = False) -> torch.Tensor:
        """SeqSharded k, v (H_kv, L, d) [or token-major (L, H_kv, d)] -> HeadSharded
        KV chunk (2, Hkl, C, dk) bf16. GQA replication happens in the pack's head map."""
        d_hp = self.par.d_hp
        send = self._new(name + ".send", (d_hp, 2, self.Hkl, self.L, dk), torch.bfloat16, fresh and d_hp == 1)
        if token_major and k.shape[-1] == dk and k.dtype == v.dtype == torch.bfloat16 \
                and k.stride(-1) == 1 and v.stride(-1) == 1:
            rows = send.view(d_hp * 2 * self.Hkl, self.L, dk).transpose(0, 1)
            K.copy_rows(k, rows, self._smap, self._dmap_k)
            K.copy_rows(v, rows, self._smap, self._dmap_v)
        else:
            if token_major:
                k, v = k.transpose(0, 1), v.transpose(0, 1)
            k, v = K.pad_dim(k, dk), K.pad_dim(v, dk)
            K.gather_blocks(k, self._smap, send, self._dmap_k)
            K.gather_blocks(v, self._smap, send, self._dmap_v)
        if d_hp == 1:
            return send.view(2, self.Hkl, self.C, dk)
        recv = self._xchg(send, name)
        out = self._new(name, (2, self.Hkl, self.C, dk), torch.bfloat16, fresh)
        return K.permute_blocks(recv, d_hp, 2 * self.Hkl, out=out)

    def _gather(self, x: torch.Tensor, name: str, fresh: bool = False) -> torch.Tensor:
        """HeadSharded (B, C, e) -> SeqSharded (d_hp*B, L, e), any dtype.
        fresh=True returns newly allocated memory (results handed to the caller)."""
        d_hp = self.par.d_hp
        if d_hp == 1:
            return x.clone() if fresh else x
        B = x.shape[0]
        send = self._buf(name + ".send", (d_hp, B) + (self.L,) + tuple(x.shape[2:]), x.dtype)
        K.permute_blocks(x.contiguous(), B, d_hp, out=send)
        recv = self._xchg(send, name)
        if fresh:
            recv = recv.clone()
        return recv.view((d_hp * B, self.L) + tuple(x.shape[2:]))

    def _gather_f32(self, x: torch.Tensor, name: str, fresh: bool = False) -> torch.Tensor:
        """HeadSharded fp32 (B, C, e) -> SeqSharded bf16 (d_hp*B, L, e): the
        fp32 -> bf16 rounding is fused into the all-to-all pack (one pass)."""
        d_hp = self.par.d_hp
        B = x.shape[0]
        if d_hp == 1:
            return K.permute_to_bf16(x, 1, 1, out=self._new(name + ".bf16", x.shape, torch.bfloat16, fresh))
        send = self._buf(name + ".send", (d_hp, B, self.L) + tuple(x.shape[2:]), torch.bfloat16)
        K.permute_to_bf16(x, B, d_hp, out=send)
        recv = self._xchg(send, name)
        if fresh:
            recv = recv.clone()
        return recv.view((d_hp * B, self.L) + tuple(x.shape[2:]))

    def _gather_dq(self, acc: torch.Tensor, name: str, fresh: bool = False) -> torch.Tensor:
        """Transposed fp32 dQ accumulator (Hl, 128, C_pad) -> SeqSharded bf16 dQ
        (d_hp*Hl, L, 128); the transpose + rounding is the all-to-all pack."""
        d_hp, Hl = self.par.d_hp, acc.shape[0]
        if d_hp == 1:
            out = self._new(name + ".bf16", (1, Hl, self.C, self.bd), torch.bfloat16, fresh)
            return K.dqt_to_bf16(acc, self.C, 1, out=out)[0]
        send = self._buf(name + ".send", (d_hp, Hl, self.L, self.bd), torch.bfloat16)
        K.dqt_to_bf16(acc, self.C, d_hp, out=send)
        recv = self._xchg(send, name)
        if fresh:
            recv = recv.clone()
        return recv.view(d_hp * Hl, self.L, self.bd)

    def _to_layout(self, x: torch.Tensor, token_major: bool) -> torch.Tensor:
        """Head-major (H, L, e>=d) result -> caller's layout, head dim d, fresh memory."""
        if not token_major:
            return x[..., :self.d] if x.shape[-1] != self.d else x
        out = torch.empty((x.shape[1], x.shape[0], self.d), dtype=x.dtype, device=x.device)
        src = x[..., :self.d] if x.shape[-1] != self.d else x
        if (self.d * x.element_size()) % 16 == 0 and src.stride(-1) == 1:
            K.copy_rows(src.transpose(0, 1), out)
        else:
            out.copy_(src.transpose(0, 1))
        return out

    def _p2p(self, group, send_t, to, recv_t, frm):
        if not self.comm_enabled:
            return None
        ops = [dist.P2POp(dist.isend, send_t, to, group), dist.P2POp(dist.irecv, recv_t, frm, group)]
        return dist.batch_isend_irecv(ops)

    @staticmethod
    def _wait(works):
        """Stream-order the current stream after NCCL works / CUDA events."""
        for wk in works or ():
            if wk is None:
                continue
            if isinstance(wk, torch.cuda.Event):
                torch.cuda.current_stream().wait_event(wk)
            else:
                wk.wait()

    # ------------------------------------------------------------ ring forward
    def _ring_forward(self, qh, kv_own, out_h, lse, mark: bool = True):
        d_cp, w = self.par.d_cp, self.par.inner_ring
        qplan = self.plans[self.cp]
        kd = qh.shape[-1]
        if d_cp == 1:
            K.fwd_chunk(qh, kv_own[0], kv_own[1], qplan, self.plans[self.cp], self.causal, self.scale,
                        lse, None, out_h)
            if mark:
                self._mark("fwd.step0")
            return
        acc = self._buf("fwd.acc", (qh.shape[0], self.C, kd), torch.float32)
        inner = [self._buf(f"kv.in{i}", kv_own.shape, kv_own.dtype) for i in range(2)]
        outer = [self._buf(f"kv.out{i}", kv_own.shape, kv_own.dtype) for i in range(2)]
        cur, first = kv_own, kv_own
        w_in = w_out = None
        n_out = 0
        for s, step in enumerate(self.steps):
            t = step.inner
            o = step.outer
            if t == 0 and o + 1 < d_cp // w:
                nxt_outer = outer[n_out % 2]
                n_out += 1
                w_out = self._p2p(self.ring_outer, first, self.outer_to, nxt_outer, self.outer_from)
            if t + 1 < w:
                nxt_inner = inner[(t + 1) % 2]
                w_in = self._p2p(self.ring_inner, cur, self.inner_to, nxt_inner, self.inner_from)
            last = s == d_cp - 1
            K.fwd_chunk(qh, cur[0], cur[1], qplan, self.plans[step.source], self.causal, self.scale, lse, acc,
                        out_h if last else None, merge=s > 0)
            if mark:
                self._mark(f"fwd.step{s}")
            if t + 1 < w:
                self._wait(w_in)
                cur = nxt_inner
            elif not last:
                self._wait(w_out)
                cur = first = nxt_outer

    # ------------------------------------------------------------ ring backward
    def _ring_backward(self, qh, kv_own, doh, lse2, delta, dq_acc, mark: bool = True):
        d_cp, w = self.par.d_cp, self.par.inner_ring
        qplan = self.plans[self.cp]
        shape = (2, kv_own.shape[1], self.C, self.bd)
        if d_cp == 1:
            dkv = self._buf("bwd.dkv_home", shape, torch.float32)
            K.bwd_chunk(qh, kv_own[0], kv_own[1], doh, qplan, self.plans[self.cp], lse2, delta, dq_acc,
                        dkv[0], dkv[1], False, self.causal, self.scale)
            if mark:
                self._mark("bwd.step0")
            return dkv
        part = self._buf("bwd.part", shape, torch.float32)
        acc = [self._buf(f"bwd.acc{i}", shape, torch.float32) for i in range(2)]
        # The home rank adds nothing after the last hop and rounds to bf16 anyway:
        # without GQA replicas (summed in fp32 after the gather) the last hop
        # carries bf16 — bit-identical, half the bytes of the exposed hop.
        home_bf16 = self.rep == 1
        home = self._buf("bwd.dkv_home", shape, torch.bfloat16 if home_bf16 else torch.float32)
        inner = [self._buf(f"kvb.in{i}", kv_own.shape, kv_own.dtype) for i in range(2)]
        outer = [self._buf(f"kvb.out{i}", kv_own.shape, kv_own.dtype) for i in range(2)]
        cur, first = kv_own, kv_own
        w_in = w_out = w_dkv = None
        n_out = 0
        for s, step in enumerate(self.steps):
            t, o = step.inner, step.outer
            if t == 0 and o + 1 < d_cp // w:
                nxt_outer = outer[n_out % 2]
                n_out += 1
                w_out = self._p2p(self.ring_outer, first, self.outer_to, nxt_outer, self.outer_from)
            if t + 1 < w:
                nxt_inner = inner[(t + 1) % 2]
                w_in = self._p2p(self.ring_inner, cur, self.inner_to, nxt_inner, self.inner_from)
            # partial dK/dV of the visiting chunk (no dependency on the travelling accumulator)
            tgt = acc[s % 2] if s == 0 else part
            K.bwd_chunk(qh, cur[0], cur[1], doh, qplan, self.plans[step.source], lse2, delta, dq_acc,
                        tgt[0], tgt[1], False, self.causal, self.scale)
            if s > 0:
                self._wait(w_dkv)            # accumulator of this chunk arrived in acc[s % 2]
                K.add_(acc[s % 2], part)     # K4: accumulate ...
            if mark:
                self._mark(f"bwd.step{s}")
            # ... and forward: next consumer is (r, p+1) inside an outer step, (r+1, p+1) across
            last = s == d_cp - 1
            dst = home if last else acc[(s + 1) % 2]
            if dkv_hop(s, d_cp, w) == "inner":
                to, frm = self.inner_to, self.inner_from
            else:
                to, frm = self.diag_to, self.diag_from
            src = acc[s % 2]
            if last and home_bf16:
                src = K.to_bf16(src, self._buf("bwd.dkv_send", shape, torch.bfloat16))
            w_dkv = self._p2p(self.ring_dkv, src, to, dst, frm)
            if t + 1 < w:
                self._wait(w_in)
                cur = nxt_inner
            elif not last:
                self._wait(w_out)
                cur = first = nxt_outer
        self._wait(w_dkv)
        return home

    # ------------------------------------------------------------ public
    def _check_inputs(self, q, k, v, token_major):
        H, Hkv, L, d = self.model.heads, self.model.kv_heads, self.L, self.d
        want_q, want_kv = ((L, H, d), (L, Hkv, d)) if token_major else ((H, L, d), (Hkv, L, d))
        if tuple(q.shape) != want_q:
            raise ValueError(f"q must be {want_q}, got {tuple(q.shape)}")
        if tuple(k.shape) != want_kv or tuple(v.shape) != want_kv:
            raise ValueError(f"k/v must be {want_kv}")

    @staticmethod
    def _layout(layout: str) -> bool:
        if layout not in ("hld", "lhd"):
            raise ValueError(f"layout must be 'hld' or 'lhd', got {layout!r}")
        return layout == "lhd"

    def _scatter_grouped(self, q, k, v, tm: bool):
        """Issue every head group's q/kv all-to-all (NCCL stream) up front.
        Returns (qh, kvh, waits): qh (Hl, C, d) and kvh (ng, 2, Hk_g, C, d) are
        filled group by group by finish(g), which stream-orders on the group's
        transfer and unpacks it."""
        d_hp, dk = self.par.d_hp, self.bd
        qh = torch.empty((self.Hl, self.C, dk), dtype=torch.bfloat16, device=self.device)
        kvh = torch.empty((self.ng, 2, self.Hk_g, self.C, dk), dtype=torch.bfloat16, device=self.device)
        pend = []
        for g in range(self.ng):
            sq, skv = self._send_q_g(q, g, "q", tm), self._send_kv_g(k, v, g, tm)
            rq, wq = self._xchg(sq, "q", g, wait=False)
            rkv, wkv = self._xchg(skv, "kv", g, wait=False)
            pend.append((rq, rkv, wq, wkv))

        def finish(g):
            rq, rkv, wq, wkv = pend[g]
            self._wait([wq, wkv])
            lo = g * self.Hq_g
            K.permute_blocks(rq, d_hp, self.Hq_g, out=qh[lo:lo + self.Hq_g])
            K.permute_blocks(rkv, d_hp, 2 * self.Hk_g, out=kvh[g])
        return qh, kvh, finish

    def scatter_inputs(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: str = "hld"):
        """SeqSharded q, k, v -> HeadSharded (qh, kvh) in memory they own (ref
        seq_alltoall_scatter + kv_replicate, sharding.py:109-152); kvh is
        (ng, 2, Hk_g, C, d), head group major."""
        tm = self._layout(layout)
        self._check_inputs(q, k, v, tm)
        if self.ng > 1:
            qh, kvh, finish = self._scatter_grouped(q, k, v, tm)
            for g in range(self.ng):
                finish(g)
            return qh, kvh
        kd = self.kd
        return (self._scatter_q(q, "q", kd, tm, fresh=True),
                self._scatter_kv(k, v, "kv", kd, tm, fresh=True).unsqueeze(0))

    def _out_tensor(self, heads: int, tm: bool) -> torch.Tensor:
        shape = (self.L, heads, self.d) if tm else (heads, self.L, self.d)
        return torch.empty(shape, dtype=torch.bfloat16, device=self.device)

    def gather_output(self, out_h: torch.Tensor, layout: str = "hld") -> torch.Tensor:
        """HeadSharded O -> SeqSharded O in the caller's layout (ref seq_alltoall_gather)."""
        tm = self._layout(layout)
        if self.ng > 1:
            out = self._out_tensor(self.model.heads, tm)
            for g in range(self.ng):
                r = self._gather_g(out_h[g * self.Hq_g:(g + 1) * self.Hq_g], "out", g, "bf16")
                self._unpack_g(*r, self._qmap[g], out, tm)
            return out
        return self._to_layout(self._gather(out_h, "out", fresh=not tm), tm)

    def _gather_g(self, x: torch.Tensor, name: str, g: int, src: str, wait: bool = True):
        """Head group g of a HeadSharded tensor -> (recv [d_hp][Hn][L][d] bf16, Work).
        src: "bf16" (Hn, C, d), "f32" (Hn, C, d) fp32, "dqt" transposed dQ accumulator."""
        d_hp, Hn = self.par.d_hp, x.shape[0]
        send = self._buf(f"{name}.gsend{g}", (d_hp, Hn, self.L, self.bd if src == "dqt" else x.shape[-1]),
                         torch.bfloat16)
        if src == "dqt":
            K.dqt_to_bf16(x, self.C, d_hp, out=send)
        elif src == "f32":
            K.permute_to_bf16(x, Hn, d_hp, out=send)
        else:
            K.permute_blocks(x, Hn, d_hp, out=send)
        recv, w = self._xchg(send, name, g, wait=False)
        if wait:
            self._wait([w])
            return (recv,)
        return recv, w

    def forward_with_state(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: str = "hld"):
        """forward() returning (out, state); state = (qh, kvh, out_h, lse) owns its
        memory, so any number of calls (layers) can be in flight before their backward."""
        tm = self._layout(layout)
        self._check_inputs(q, k, v, tm)
        self.times.clear()
        self._mark("fwd.start")
        kd = self.kd
        if self.ng > 1:
            # pipelined: group g's ring overlaps group g+1's input exchange and
            # group g-1's output exchange
            qh, kvh, finish = self._scatter_grouped(q, k, v, tm)
            out_h = torch.empty((self.Hl, self.C, kd), dtype=torch.bfloat16, device=self.device)
            lse = torch.empty((self.Hl, self.C), dtype=torch.float32, device=self.device)
            out = self._out_tensor(self.model.heads, tm)
            pend = []
            for g in range(self.ng):
                finish(g)
                if g == 0:
                    self._mark("fwd.a2a_in")
                sl = slice(g * self.Hq_g, (g + 1) * self.Hq_g)
                self._ring_forward(qh[sl], kvh[g], out_h[sl], lse[sl], mark=g == self.ng - 1)
                pend.append(self._gather_g(out_h[sl], "out", g, "bf16", wait=False))
            for g, (recv, w) in enumerate(pend):
                self._wait([w])
                self._unpack_g(recv, self._qmap[g], out, tm)
            self._mark("fwd.a2a_out")
            return out, (qh, kvh, out_h, lse)
        qh = self._scatter_q(q, "q", kd, tm, fresh=True)
        kvh = self._scatter_kv(k, v, "kv", kd, tm, fresh=True)
        self._mark("fwd.a2a_in")
        out_h = torch.empty((self.Hl, self.C, kd), dtype=torch.bfloat16, device=self.device)
        lse = torch.empty((self.Hl, self.C), dtype=torch.float32, device=self.device)
        self._ring_forward(qh, kvh, out_h, lse)
        out = self._gather(out_h, "out", fresh=not tm)
        self._mark("fwd.a2a_out")
        state = _State((qh, kvh.unsqueeze(0), out_h, lse))
        if qh.data_ptr() == q.data_ptr():
            state.guard = (q, q._version)
        return self._to_layout(out, tm), state

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: str = "hld") -> torch.Tensor:
        """This rank's SeqSharded chunk -> SeqSharded output, bf16.

        layout "hld": q (H, L, d), k/v (H_kv, L, d) head-major (the reference's
        DenseTensor.values); "lhd": token-major (L, H, d) / (L, H_kv, d), strided
        views (e.g. slices of a fused QKV projection output) accepted as is.
        Output in the same layout. The state for backward() is kept on the op
        (last call); autograd use goes through Attn2DFunction, which keeps one
        state per call."""
        out, self.saved = self.forward_with_state(q, k, v, layout)
        return out

    def backward(self, dout: torch.Tensor, layout: str = "hld", state=None):
        """SeqSharded dout -> (dq, dk, dv) SeqSharded, bf16, in the given layout.
        `state` is a forward_with_state() state (default: the last forward())."""
        tm = self._layout(layout)
        state = state if state is not None else self.saved
        if state is None:
            raise RuntimeError("backward called before forward")
        qh, kvh, out_h, lse = state
        guard = getattr(state, "guard", None)
        if guard is not None and guard[0]._version != guard[1]:
            raise RuntimeError("q was modified in place between forward and backward (the saved state aliases it "
                               "when d_hp = 1); clone q before modifying it")
        self._mark("bwd.start")
        bd = self.bd
        if self.ng > 1:
            return self._backward_grouped(dout, tm, qh, kvh, out_h, lse)
        kvh = kvh[0]
        if self.kd != bd:  # head dim <= 64: the backward kernel runs at 128 (exact zero padding)
            qh, kvh, out_h = K.pad_dim(qh, bd), K.pad_dim(kvh, bd), K.pad_dim(out_h, bd)
        out_b = out_h
        doh = self._scatter_q(dout, "do", bd, tm)
        self._mark("bwd.a2a_in")
        lse2, delta = K.bwd_preprocess(out_b, doh, lse)
        dq_acc = self._buf("dq_acc", (self.Hl, bd, self.C_pad), torch.float32)
        dq_acc.zero_()
        dkv = self._ring_backward(qh, kvh, doh, lse2, delta, dq_acc)
        self._mark("bwd.ring")
        dq = self._gather_dq(dq_acc, "dq", fresh=not tm)
        self._mark("bwd.a2a_dq")
        if self.rep == 1:
            # one all-to-all per tensor: each receive buffer is already (H_kv, L, e);
            # dkv is bf16 when it arrived by the ring's last hop, fp32 straight from the kernel
            gather = self._gather if dkv.dtype == torch.bfloat16 else self._gather_f32
            dk, dv = gather(dkv[0], "dk", fresh=not tm), gather(dkv[1], "dv", fresh=not tm)
        else:  # GQA replicas: gather fp32, sum the Ĥ/H_kv copies, then round once
            dk = K.to_bf16(K.sum_replicas(self._gather(dkv[0], "dk32"), self.rep))
            dv = K.to_bf16(K.sum_replicas(self._gather(dkv[1], "dv32"), self.rep))
        self._mark("bwd.a2a_out")
        return self._to_layout(dq, tm), self._to_layout(dk, tm), self._to_layout(dv, tm)

    def _backward_grouped(self, dout, tm, qh, kvh, out_h, lse):
        """Pipelined backward: every group's dO all-to-all is issued up front;
        group g's gradient gather (fp32 -> bf16 fused into the pack) runs on
        NCCL's stream while group g+1's ring backward computes."""
        d_hp, bd = self.par.d_hp, self.bd
        pend_in = []
        for g in range(self.ng):
            sd = self._send_q_g(dout, g, "do", tm)
            pend_in.append(self._xchg(sd, "do", g, wait=False))
        dq = self._out_tensor(self.model.heads, tm)
        dk = self._out_tensor(self.H_rep, tm)
        dv = self._out_tensor(self.H_rep, tm)
        pend_out = []
        for g in range(self.ng):
            rd, w = pend_in[g]
            self._wait([w])
            doh = self._buf("doh", (self.Hq_g, self.C, bd), torch.bfloat16)
            K.permute_blocks(rd, d_hp, self.Hq_g, out=doh)
            if g == 0:
                self._mark("bwd.a2a_in")
            sl = slice(g * self.Hq_g, (g + 1) * self.Hq_g)
            lse2, delta = K.bwd_preprocess(out_h[sl], doh, lse[sl])
            dq_acc = self._buf("dq_acc", (self.Hq_g, bd, self.C_pad), torch.float32)
            dq_acc.zero_()
            dkv = self._ring_backward(qh[sl], kvh[g], doh, lse2, delta, dq_acc, mark=g == self.ng - 1)
            for name, src, dst, hmap in (("dq", dq_acc, dq, self._qmap[g]), ("dk", dkv[0], dk, self._kmap[g]),
                                         ("dv", dkv[1], dv, self._kmap[g])):
                kind = "dqt" if name == "dq" else ("bf16" if src.dtype == torch.bfloat16 else "f32")
                recv, w = self._gather_g(src, name, g, kind, wait=False)
                pend_out.append((recv, w, hmap, dst))
        self._mark("bwd.ring")
        for recv, w, hmap, dst in pend_out:
            self._wait([w])
            self._unpack_g(recv, hmap, dst, tm)
        self._mark("bwd.a2a_out")
        return dq, dk, dv

    def flops(self) -> float:
        """Algorithmic fwd+bwd FLOPs of the whole layer (all ranks): 3.5 x 4 S^2 H d x (1/2 if causal)."""
        S, H = self.model.seq_len, self.model.heads
        return 3.5 * 4.0 * S * S * H * self.d * (0.5 if self.causal else 1.0)


class Attn2DFunction(torch.autograd.Function):
    """autograd wrapper: saves O and LSE (selective-checkpoint friendly), no recompute of attention."""

    @staticmethod
    def forward(ctx, q, k, v, op: Attn2D, layout: str = "hld"):
        ctx.op, ctx.layout = op, layout
        out, ctx.state = op.forward_with_state(q, k, v, layout)
        return out

    @staticmethod
    def backward(ctx, dout):
        dq, dk, dv = ctx.op.backward(dout.contiguous() if ctx.layout == "hld" else dout, ctx.layout, ctx.state)
        ctx.state = None
        return dq, dk, dv, None, None


def shard_global(x: torch.Tensor, op: Attn2D) -> torch.Tensor:
    """This rank's SeqSharded chunk of a global (H, S, d) tensor (ref shard_sequence,
    sharding.py:56-79): the 128-bit gather_tokens kernel."""
    return K.gather_tokens(x, op.seq_pos)


def unshard_global(chunks: list[torch.Tensor], op: Attn2D) -> torch.Tensor:
    """Reassemble global (H, S, d) from all ranks' SeqSharded chunks (ref unshard,
    sharding.py:91-106): one gather_tokens scatter per chunk."""
    S = op.model.seq_len
    out = torch.empty((chunks[0].shape[0], S) + tuple(chunks[0].shape[2:]), dtype=chunks[0].dtype,
                      device=chunks[0].device)
    for r, c in enumerate(chunks):
        hp, cp = op.grid.coords_of(r)
        K.gather_tokens(c, seq_positions(S, op.grid, hp, cp), out=out, scatter=True)
    return out


def positions_of_rank(op: Attn2D, rank: int) -> np.ndarray:
    hp, cp = op.grid.coords_of(rank)
    return seq_positions(op.model.seq_len, op.grid, hp, cp)
