"""torch-facing wrappers over the C ABI (device memory, streams, padding).

Every function here launches CUDA work through ``libattn2d_sm100.so`` on the
current torch stream; none has a CPU path. Tensor layout is head-major
``[H][T][D]`` (the reference's DenseTensor.values, oracle.py:15-34).
"""

from __future__ import annotations

import math

import torch

from . import _lib

BF16 = torch.bfloat16
FWD_DIMS = (64, 128)
BWD_DIMS = (64, 128)
BWD_DIM = 128  # the native runtime's head dim
BWD_QSLICE = 2048 * 64  # query rows per fa_bwd launch (capi.cu a2d_fa_bwd_chunk)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _check_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("tensor must live on a CUDA device")


def fwd_dim(d: int) -> int:
    """Kernel head dim for a true head dim d (zero padding, exact)."""
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise ValueError(f"head_dim {d} > 128 not supported")


def pad_dim(x: torch.Tensor, dk: int) -> torch.Tensor:
    """bf16, contiguous, last dim zero-padded to dk (QK^T and PV unchanged)."""
    x = x.to(BF16)
    if x.shape[-1] != dk:
        x = torch.nn.functional.pad(x, (0, dk - x.shape[-1]))
    return x.contiguous()


def tile_bounds(pos: torch.Tensor, tile: int) -> torch.Tensor:
    """[ceil(T/tile), 2] int32 (min, max) of positions per tile."""
    _check_cuda(pos)
    pos = pos.to(torch.int32).contiguous()
    n = (pos.numel() + tile - 1) // tile
    out = torch.empty((max(n, 1), 2), dtype=torch.int32, device=pos.device)
    _lib.call("a2d_tile_bounds", pos.data_ptr(), pos.numel(), tile, out.data_ptr(), _stream())
    return out


class ChunkPlan:
    """Positions + tile bounds of one chunk, cached for reuse across steps."""

    def __init__(self, pos: torch.Tensor):
        self.pos = pos.to(torch.int32).contiguous()
        self.b128 = tile_bounds(self.pos, 128)
        self.b64 = tile_bounds(self.pos, 64)

    @property
    def T(self) -> int:
        return self.pos.numel()


def fwd_chunk(q, k, v, qp: ChunkPlan, kp: ChunkPlan, causal: bool, scale: float,
              lse: torch.Tensor, acc_o: torch.Tensor | None = None,
              out: torch.Tensor | None = None, merge: bool = False) -> None:
    """One ring step forward (K1 + fused K2). q/k/v bf16 [H|Hkv][T][D], D in {64,128}."""
    _check_cuda(q, k, v)
    H, Tq, D = q.shape
    Hkv, Tk, _ = k.shape
    if D not in FWD_DIMS:
        raise ValueError(f"kernel head dim must be 64 or 128, got {D}")
    for t in (q, k, v):
        if t.dtype != BF16 or not t.is_contiguous():
            raise ValueError("q/k/v must be contiguous bf16")
    if k.shape != v.shape:
        raise ValueError("K and V shapes differ")
    _lib.call("a2d_fa_fwd_chunk", q.data_ptr(), k.data_ptr(), v.data_ptr(), qp.pos.data_ptr(),
              kp.pos.data_ptr(), qp.b128.data_ptr(), kp.b128.data_ptr(), H, Hkv, Tq, Tk, D,
              int(causal), float(scale), int(merge), lse.data_ptr(),
              None if acc_o is None else acc_o.data_ptr(),
              None if out is None else out.data_ptr(), _stream())


def bwd_preprocess(o: torch.Tensor, dout: torch.Tensor, lse: torch.Tensor):
    """(lse2, delta) fp32 [H][Tq_pad64]."""
    H, Tq, D = o.shape
    tp = (Tq + 63) // 64 * 64
    lse2 = torch.empty((H, tp), dtype=torch.float32, device=o.device)
    delta = torch.empty((H, tp), dtype=torch.float32, device=o.device)
    _lib.call("a2d_bwd_preprocess", o.data_ptr(), dout.data_ptr(), lse.data_ptr(), H, Tq, D,
              lse2.data_ptr(), delta.data_ptr(), _stream(), nbytes=H * Tq * (4 * D + 4) + H * tp * 8)
    return lse2, delta


def dq_acc_t(H: int, T: int, device, D: int = BWD_DIM) -> torch.Tensor:
    """Zeroed transposed dQ accumulator [H][D][round_up(T, 64)] fp32 (bwd_chunk's dq_acc)."""
    return torch.zeros((H, D, (T + 63) // 64 * 64), dtype=torch.float32, device=device)


def dq_from_acc(acc: torch.Tensor, T: int) -> torch.Tensor:
    """fp32 [H][T][128] view of a transposed accumulator (tests / the global-view API)."""
    return acc[:, :, :T].transpose(1, 2)


def dqt_to_bf16(acc: torch.Tensor, T: int, A: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """bf16 dQ out of the transposed accumulator: out[a][h][l][:] = acc[h][:][a*L + l], L = T/A."""
    H, D = acc.shape[0], acc.shape[1]
    if out is None:
        out = torch.empty((A, H, T // A, D), dtype=BF16, device=acc.device)
    _lib.call("a2d_dqt_to_bf16_d", acc.data_ptr(), out.data_ptr(), H, T, acc.shape[2], A, D, _stream(),
              nbytes=H * T * D * 6)
    return out


def bwd_chunk(q, k, v, dout, qp: ChunkPlan, kp: ChunkPlan, lse2, delta, dq_acc, dk, dv,
              accumulate_kv: bool, causal: bool, scale: float) -> None:
    """One ring step backward (K3). q/k/v/dout bf16 D in {64, 128}; dk/dv fp32 [H_kv][Tk][D];
    dq_acc fp32 TRANSPOSED [H][D][round_up(Tq, 64)] (see dq_acc_t / dqt_to_bf16)."""
    H, Tq, D = q.shape
    Hkv, Tk, _ = k.shape
    n_launch = max(1, -(-Tq // BWD_QSLICE)) if Tk > 0 else 0  # the C ABI slices long query chunks
    if D not in BWD_DIMS:
        raise ValueError("backward kernel head dim must be 64 or 128")
    if dq_acc.shape != (H, D, (Tq + 63) // 64 * 64) or dq_acc.dtype != torch.float32:
        raise ValueError("dq_acc must be the transposed fp32 accumulator [H][D][round_up(Tq, 64)]")
    _lib.call("a2d_fa_bwd_chunk", q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(),
              qp.pos.data_ptr(), kp.pos.data_ptr(), qp.b64.data_ptr(), kp.b128.data_ptr(),
              lse2.data_ptr(), delta.data_ptr(), dq_acc.data_ptr(), dk.data_ptr(), dv.data_ptr(),
              int(accumulate_kv), H, Hkv, Tq, Tk, D, int(causal), float(scale), _stream(), launches=n_launch)


def merge_(acc_o, acc_lse, blk_o, blk_lse) -> None:
    """In-place block_update of fp32 (acc_o, acc_lse) with (blk_o, blk_lse)."""
    d = acc_o.shape[-1]
    rows = acc_o.numel() // d
    blk = blk_o.contiguous().float()
    _lib.call("a2d_merge", acc_o.data_ptr(), acc_lse.data_ptr(), blk.data_ptr(), blk_lse.data_ptr(), rows, d,
              _stream(), nbytes=rows * (12 * d + 12))


def permute_blocks(src: torch.Tensor, A: int, B: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[b][a] = src[a][b] with src viewed as [A][B][blk] (bit-exact byte move)."""
    src = src.contiguous()
    if out is None:
        out = torch.empty_like(src)
    blk = src.numel() * src.element_size() // max(A * B, 1)
    _lib.call("a2d_permute_blocks", src.data_ptr(), out.data_ptr(), A, B, blk, _stream(), nbytes=2 * A * B * blk)
    return out


def gather_blocks(src: torch.Tensor, index: torch.Tensor, out: torch.Tensor,
                  dst_index: torch.Tensor | None = None, block_elems: int | None = None) -> torch.Tensor:
    """out[dst_index[i] or i] = src[index[i]] over blocks (default: leading-dim slices)."""
    if block_elems is None:
        block_elems = src[0].numel()
    blk = block_elems * src.element_size()
    idx = index.to(device=src.device, dtype=torch.int32).contiguous()
    didx = None if dst_index is None else dst_index.to(device=src.device, dtype=torch.int32).contiguous()
    _lib.call("a2d_gather_blocks", src.data_ptr(), out.data_ptr(), idx.data_ptr(),
              None if didx is None else didx.data_ptr(), idx.numel(), blk, _stream(), nbytes=2 * idx.numel() * blk)
    return out


def copy_rows(src: torch.Tensor, dst: torch.Tensor, src_map: torch.Tensor | None = None,
              dst_map: torch.Tensor | None = None) -> torch.Tensor:
    """dst[t, dmap(h), :] = src[t, smap(h), :] for 3-D (T, H, row) views with any
    (t, h) strides and a contiguous last dim — e.g. token-major <-> head-major
    (pass ``x.transpose(0, 1)``) or a head slice of a fused QKV buffer."""
    if src.dim() != 3 or dst.dim() != 3:
        raise ValueError("copy_rows expects 3-D (T, H, row) views")
    if src.stride(2) != 1 or dst.stride(2) != 1 or src.dtype != dst.dtype:
        raise ValueError("copy_rows needs a contiguous, same-dtype last dimension")
    n_t = src.shape[0]
    n_h = (src_map.numel() if src_map is not None else src.shape[1])
    es = src.element_size()
    row = src.shape[2] * es
    dev = src.device
    sm = None if src_map is None else src_map.to(device=dev, dtype=torch.int32).contiguous()
    dm = None if dst_map is None else dst_map.to(device=dev, dtype=torch.int32).contiguous()
    _lib.call("a2d_copy_rows", src.data_ptr(), dst.data_ptr(), n_t, n_h, src.stride(0) * es, src.stride(1) * es,
              dst.stride(0) * es, dst.stride(1) * es, row, None if sm is None else sm.data_ptr(),
              None if dm is None else dm.data_ptr(), _stream(), nbytes=2 * n_t * n_h * row)
    return dst


def gather_tokens(src: torch.Tensor, idx, out: torch.Tensor | None = None, scatter: bool = False,
                  out_tokens: int | None = None) -> torch.Tensor:
    """Token rows of every head (ref shard_sequence / unshard, sharding.py:56-106):
    gather out[h][t] = src[h][idx[t]], or scatter out[h][idx[t]] = src[h][t].
    src (H, S, ...) contiguous with 16-byte-multiple rows; any dtype (byte move)."""
    _check_cuda(src)
    src = src.contiguous()
    idx = torch.as_tensor(idx, device=src.device).to(torch.int32).contiguous()
    H, S = src.shape[0], src.shape[1]
    row = src[0, 0].numel() * src.element_size() if S else 16
    L = idx.numel()
    if out is None:
        n = (out_tokens if out_tokens is not None else S) if scatter else L
        out = torch.empty((H, n) + tuple(src.shape[2:]), dtype=src.dtype, device=src.device)
    if row % 16 or out.dtype != src.dtype or not out.is_contiguous():
        raise ValueError("gather_tokens needs contiguous same-dtype tensors with 16-byte-multiple rows")
    _lib.call("a2d_gather_tokens", src.data_ptr(), out.data_ptr(), idx.data_ptr(), H, S, L, out.shape[1], row,
              int(scatter), _stream(), nbytes=2 * H * L * row)
    return out


def sum_replicas(src: torch.Tensor, rep: int) -> torch.Tensor:
    """[H*rep, ...] fp32 -> [H, ...] summing consecutive copies."""
    heads = src.shape[0] // rep
    out = torch.empty((heads,) + tuple(src.shape[1:]), dtype=torch.float32, device=src.device)
    _lib.call("a2d_sum_replicas_f32", src.data_ptr(), out.data_ptr(), heads, rep, src[0].numel(), _stream(),
              nbytes=4 * (rep + 1) * heads * src[0].numel())
    return out


def to_bf16(src: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(src.shape, dtype=BF16, device=src.device)
    _lib.call("a2d_f32_to_bf16", src.data_ptr(), out.data_ptr(), src.numel(), _stream(), nbytes=6 * src.numel())
    return out


def permute_to_bf16(src: torch.Tensor, A: int, B: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[b][a] = bf16(src[a][b]) with fp32 src viewed as [A][B][blk] (convert fused into the pack)."""
    src = src.contiguous()
    if out is None:
        out = torch.empty(src.shape, dtype=BF16, device=src.device)
    blk = src.numel() // max(A * B, 1)
    _lib.call("a2d_permute_f32_to_bf16", src.data_ptr(), out.data_ptr(), A, B, blk, _stream(),
              nbytes=6 * src.numel())
    return out


def add_(dst: torch.Tensor, src: torch.Tensor) -> None:
    _lib.call("a2d_add_f32", dst.data_ptr(), src.data_ptr(), dst.numel(), _stream(), nbytes=12 * dst.numel())


def selftest_umma(a, b, v, at) -> torch.Tensor:
    c = torch.empty((4, 128, 128), dtype=torch.float32, device=a.device)
    _lib.call("a2d_selftest_umma", a.data_ptr(), b.data_ptr(), v.data_ptr(), at.data_ptr(), c.data_ptr(),
              _stream())
    return c


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
