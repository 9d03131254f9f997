"""torch face of the native SPMD runtime (C ABI a2d_ctx_create / a2d_fwd /
a2d_bwd, csrc/runtime.cu): the whole 2D-attention layer of one rank, NCCL
inside the library. Same tensors and layout as ``dist.Attn2D`` (head-major
SeqSharded chunks in zig-zag order); torch.distributed only hands the NCCL id
from rank 0 to the others."""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .config import ClusterConfig, ModelConfig, ParallelConfig, Placement, build_rank_grid, check_config


class NativeAttn2D:
    def __init__(self, model: ModelConfig, par: ParallelConfig, cluster: ClusterConfig | None = None,
                 causal: bool = True):
        check_config(model, par, cluster or ClusterConfig())
        if model.head_dim != 128:
            raise ValueError("the native runtime supports head dim 128")
        self.model, self.par, self.causal = model, par, causal
        self.grid = build_rank_grid(par, cluster or ClusterConfig())
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if self.world != par.d_hp * par.d_cp:
            raise ValueError(f"world size {self.world} != d_hp*d_cp = {par.d_hp * par.d_cp}")
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.call("a2d_nccl_unique_id", ctypes.addressof(uid), 128)
        box = [uid.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = ctypes.create_string_buffer(box[0], 128)
        self._uid = uid
        self._ctx = ctypes.c_void_p()
        placement = 0 if par.placement is Placement.HEAD_FIRST else 1
        _lib.call("a2d_ctx_create", ctypes.addressof(uid), self.rank, self.world, par.d_hp, par.d_cp,
                  par.inner_ring, placement, model.heads, model.kv_heads, model.head_dim, model.seq_len,
                  int(causal), ctypes.addressof(self._ctx))
        self.L = model.seq_len // self.world
        nb = ctypes.c_int64()
        _lib.call("a2d_saved_bytes", self._ctx, ctypes.addressof(nb))
        self.saved_bytes = int(nb.value)
        self.saved = None  # state of the last forward() (forward_with_state returns its own)
        tr = ctypes.c_int32()
        _lib.call("a2d_ctx_transport", self._ctx, ctypes.addressof(tr))
        self.transport = "symm" if tr.value else "nccl"

    def _empty(self, heads: int, like: torch.Tensor) -> torch.Tensor:
        return torch.empty((heads, self.L, self.model.head_dim), dtype=torch.bfloat16, device=like.device)

    def forward_with_state(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
        """(out, state): state is a caller-owned device buffer holding this
        call's HeadSharded Q, K/V, output and LSE, so any number of forwards
        can be in flight before their backwards (stateless context)."""
        m = self.model
        for t, h in ((q, m.heads), (k, m.kv_heads), (v, m.kv_heads)):
            if tuple(t.shape) != (h, self.L, m.head_dim) or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise ValueError(f"expected contiguous bf16 ({h}, {self.L}, {m.head_dim}), got {tuple(t.shape)}")
        out = self._empty(m.heads, q)
        state = torch.empty(self.saved_bytes, dtype=torch.uint8, device=q.device)  # caching allocator: 512-B aligned
        _lib.call("a2d_fwd", self._ctx, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), state.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        return out, state

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        out, self.saved = self.forward_with_state(q, k, v)
        return out

    def backward(self, dout: torch.Tensor, state: torch.Tensor | None = None):
        """(dq, dk, dv) of the forward whose state is given (default: the last forward())."""
        m = self.model
        state = self.saved if state is None else state
        if state is None:
            raise RuntimeError("backward called before forward")
        dout = dout.to(torch.bfloat16).contiguous()
        dq, dk, dv = self._empty(m.heads, dout), self._empty(m.kv_heads, dout), self._empty(m.kv_heads, dout)
        _lib.call("a2d_bwd", self._ctx, state.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                  dv.data_ptr(), torch.cuda.current_stream().cuda_stream)
        return dq, dk, dv

    @property
    def comm_enabled(self) -> bool:
        return getattr(self, "_comm", True)

    @comm_enabled.setter
    def comm_enabled(self, on: bool) -> None:
        """Measurement only (exposed communication): False skips every NCCL call."""
        self._comm = bool(on)
        _lib.call("a2d_ctx_set_comm", self._ctx, int(self._comm))

    def kernel_timing(self, enabled: bool) -> None:
        """Start (and reset) / stop CUDA-event timing of the attention kernels."""
        _lib.call("a2d_ctx_timing", self._ctx, int(enabled))

    def kernel_ms(self) -> dict:
        """Summed fwd / bwd attention-kernel milliseconds since kernel_timing(True)."""
        f, b = ctypes.c_float(), ctypes.c_float()
        nf, nb = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("a2d_ctx_kernel_ms", self._ctx, ctypes.addressof(f), ctypes.addressof(b), ctypes.addressof(nf),
                  ctypes.addressof(nb))
        return {"fwd_ms": f.value, "bwd_ms": b.value, "n_fwd": nf.value, "n_bwd": nb.value}

    def sync(self, timeout_s: float = 600.0) -> None:
        """Wait for this rank's queued layer work, polling NCCL for asynchronous
        errors; raises (and aborts the communicators) on an error or timeout."""
        _lib.call("a2d_sync", self._ctx, torch.cuda.current_stream().cuda_stream, int(timeout_s * 1000))

    def lse_of(self, state: torch.Tensor) -> torch.Tensor:
        """The natural-log LSE [Hl][C] fp32 (HeadSharded) inside a saved state."""
        m, par = self.model, self.par
        C = m.seq_len // par.d_cp
        Hl = m.heads // par.d_hp
        up = lambda x: (x + 255) // 256 * 256  # noqa: E731
        from .config import replicated_kv_heads
        hkl = replicated_kv_heads(m.kv_heads, par.d_hp, m.heads) // par.d_hp
        off = up(Hl * C * 128 * 2) + up(2 * hkl * C * 128 * 2) + up(Hl * C * 128 * 2)
        return state[off:off + Hl * C * 4].view(torch.float32).view(Hl, C)
    def close(self) -> None:
        if self._ctx:
            _lib.call("a2d_ctx_destroy", self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
