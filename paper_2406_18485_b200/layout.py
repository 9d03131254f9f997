"""Token/head index maps of the 2D layout (pure integer math, host side).

The reference realises these as numpy index shuffles
(``/root/reference/pkg/src/attn2d/sharding.py``). On B200 the same maps drive
(a) the data-loader gather that produces each rank's SeqSharded chunk,
(b) the pack/unpack kernels around the head-parallel all-to-all, and
(c) the causal mask: the attention kernels never see a permutation, only the
per-token original positions of the chunk they work on.

Definitions (verified against the reference):

* zig-zag: the sequence is cut into 2*d_cp stripes of sigma = S/(2 d_cp)
  tokens; CP rank j owns stripes j and 2 d_cp-1-j (ref ``sharding.py:33-53``).
* SeqSharded: rank (i, j) holds all heads for tokens
  ``perm[j*C + i*L : j*C + (i+1)*L]`` with C = S/d_cp, L = S/d_sp
  (ref ``sharding.py:56-79``).
* HeadSharded: rank (i, j) holds heads ``[i*H'/d_hp, (i+1)*H'/d_hp)`` for the
  CP group's whole token set ``perm[j*C:(j+1)*C]`` in hp order
  (ref ``sharding.py:131-152``).
"""

from __future__ import annotations

import numpy as np

from .config import RankGrid


def zigzag_reorder(seq_len: int, d_cp: int) -> tuple[np.ndarray, np.ndarray]:
    """(perm, inv): perm[slot] = original position; inv = perm^-1."""
    if seq_len % (2 * d_cp) != 0:
        raise ValueError(f"S={seq_len} not divisible by 2*d_cp={2 * d_cp}")
    sigma = seq_len // (2 * d_cp)
    slot = np.arange(seq_len, dtype=np.int64)
    j, u = np.divmod(slot, 2 * sigma)
    stripe = np.where(u < sigma, j, 2 * d_cp - 1 - j)
    perm = stripe * sigma + (u % sigma)
    inv = np.empty_like(perm)
    inv[perm] = slot
    return perm, inv


def cp_positions(seq_len: int, d_cp: int, cp_index: int) -> np.ndarray:
    """Original positions of CP rank j's HeadSharded token set (C tokens)."""
    perm, _ = zigzag_reorder(seq_len, d_cp)
    c = seq_len // d_cp
    return perm[cp_index * c:(cp_index + 1) * c]


def seq_positions(seq_len: int, grid: RankGrid, hp_index: int,
                  cp_index: int) -> np.ndarray:
    """Original positions of rank (i, j)'s SeqSharded chunk (L tokens)."""
    if seq_len % (2 * grid.d_sp) != 0:
        raise ValueError(f"S={seq_len} not divisible by 2*d_sp={2 * grid.d_sp}")
    group = cp_positions(seq_len, grid.d_cp, cp_index)
    per = seq_len // grid.d_sp
    return group[hp_index * per:(hp_index + 1) * per]


def stripe_bases(seq_len: int, d_cp: int, cp_index: int) -> tuple[int, int, int]:
    """(base0, base1, sigma): CP chunk j = [base0, base0+sigma) ++ [base1, ...)."""
    sigma = seq_len // (2 * d_cp)
    return cp_index * sigma, (2 * d_cp - 1 - cp_index) * sigma, sigma


def head_slice(n_heads: int, d_hp: int, hp_index: int) -> slice:
    """Heads rank hp_index owns after the SeqAlltoAll scatter."""
    if n_heads % d_hp != 0:
        raise ValueError(f"{n_heads} heads not divisible by d_hp={d_hp}")
    per = n_heads // d_hp
    return slice(hp_index * per, (hp_index + 1) * per)


def replica_source_heads(kv_heads: int, replicated: int) -> np.ndarray:
    """Original KV head read for each replicated head slot.

    ``kv_replicate`` (ref ``sharding.py:109-128``) repeats every head
    ``replicated // kv_heads`` times contiguously, so slot h reads h // rep.
    The B200 pack kernel uses this map instead of materialising copies.
    """
    rep = replicated // kv_heads
    return np.arange(replicated) // rep
