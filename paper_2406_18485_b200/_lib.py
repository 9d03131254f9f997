"""ctypes binding of libattn2d_sm100.so (the C ABI in include/attn2d_sm100.h).

There is deliberately no fallback: if the library is missing or fails to
load, every op raises. The CPU oracle lives in ``oracle/`` and is test
infrastructure only.
"""

from __future__ import annotations

import ctypes
import os

LIB_PATH = os.environ.get("A2D_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                        "libattn2d_sm100.so")

_c_int, _c_i32, _c_i64, _c_f32, _vp = (ctypes.c_int, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_float, ctypes.c_void_p)

# name -> argtypes (all return int status)
SIGNATURES = {
    "a2d_tile_bounds": [_vp, _c_i64, _c_i32, _vp, _vp],
    "a2d_fa_fwd_chunk": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_i64, _c_i64,
                         _c_i32, _c_i32, _c_f32, _c_i32, _vp, _vp, _vp, _vp],
    "a2d_bwd_preprocess": [_vp, _vp, _vp, _c_i32, _c_i64, _c_i32, _vp, _vp, _vp],
    "a2d_fa_bwd_chunk": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                         _c_i32, _c_i32, _c_i32, _c_i64, _c_i64, _c_i32, _c_i32, _c_f32, _vp],
    "a2d_merge": [_vp, _vp, _vp, _vp, _c_i64, _c_i32, _vp],
    "a2d_permute_blocks": [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp],
    "a2d_gather_blocks": [_vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp],
    "a2d_sum_replicas_f32": [_vp, _vp, _c_i64, _c_i32, _c_i64, _vp],
    "a2d_gather_tokens": [_vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i32, _vp],
    "a2d_copy_rows": [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp],
    "a2d_f32_to_bf16": [_vp, _vp, _c_i64, _vp],
    "a2d_permute_f32_to_bf16": [_vp, _vp, _c_i64, _c_i64, _c_i64, _vp],
    "a2d_dqt_to_bf16": [_vp, _vp, _c_i32, _c_i64, _c_i64, _c_i32, _vp],
    "a2d_dqt_to_bf16_d": [_vp, _vp, _c_i32, _c_i64, _c_i64, _c_i32, _c_i32, _vp],
    "a2d_add_f32": [_vp, _vp, _c_i64, _vp],
    "a2d_selftest_umma": [_vp, _vp, _vp, _vp, _vp, _vp],
    "a2d_nccl_unique_id": [_vp, _c_i64],
    "a2d_ctx_create": [_vp, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i64, _c_i32,
                       _vp],
    "a2d_saved_bytes": [_vp, _vp],
    "a2d_fwd": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "a2d_bwd": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "a2d_sync": [_vp, _vp, _c_i64],
    "a2d_ctx_set_comm": [_vp, _c_i32],
    "a2d_ctx_transport": [_vp, _vp],
    "a2d_ctx_timing": [_vp, _c_i32],
    "a2d_ctx_kernel_ms": [_vp, _vp, _vp, _vp, _vp],
    "a2d_ctx_destroy": [_vp],
    "a2d_ring_plan": [_c_i32, _c_i32, _c_i32, _vp, _vp],
    "a2d_zigzag_positions": [_c_i64, _c_i32, _c_i32, _vp],
}

_lib = None


class KernelError(RuntimeError):
    """CUDA-side failure reported by the library."""


def load(path: str = LIB_PATH):
    """Load (once) and return the CDLL. Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} not built; run `python -m paper_2406_18485_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _c_int
    lib.a2d_last_error.restype = ctypes.c_char_p
    lib.a2d_last_error.argtypes = []
    lib.a2d_abi_version.restype = _c_int
    lib.a2d_launch_count.restype = ctypes.c_longlong
    lib.a2d_launch_count.argtypes = []
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernels launched so far by the library in this process (C-side counter)."""
    return int(load().a2d_launch_count())


# kernels each entry point launches (for the bench's gpu_launches accounting)
LAUNCHES = {"a2d_tile_bounds": 1, "a2d_fa_fwd_chunk": 1, "a2d_bwd_preprocess": 1, "a2d_fa_bwd_chunk": 1,
            "a2d_merge": 1, "a2d_permute_blocks": 1, "a2d_gather_blocks": 1, "a2d_sum_replicas_f32": 1,
            "a2d_f32_to_bf16": 1, "a2d_permute_f32_to_bf16": 1, "a2d_dqt_to_bf16": 1, "a2d_dqt_to_bf16_d": 1, "a2d_add_f32": 1, "a2d_selftest_umma": 1, "a2d_copy_rows": 1, "a2d_gather_tokens": 1}


class LaunchLog:
    """Counts library kernel launches; optionally brackets chosen entry points
    with CUDA events recorded on the launching (current) stream."""

    def __init__(self):
        self.enabled = False
        self.count = 0
        self.by_name: dict[str, int] = {}
        self.timed: set[str] = set()
        self.events: list = []  # (name, start_event, end_event, algorithmic bytes moved)

    def reset(self, timed=()):
        self.count = 0
        self.by_name = {}
        self.timed = set(timed)
        self.events = []


LOG = LaunchLog()


def call(name: str, *args, nbytes: int = 0, launches: int | None = None) -> None:
    """Invoke an entry point; map non-zero status to ValueError / KernelError.

    ``nbytes``: algorithmic HBM bytes the call moves (read + write of every
    element, for the bench's HBM roofline); ``launches``: kernels it launches
    when that depends on the arguments (default LAUNCHES[name])."""
    lib = load()
    ev = None
    if LOG.enabled:
        LOG.count += LAUNCHES.get(name, 0) if launches is None else launches
        LOG.by_name[name] = LOG.by_name.get(name, 0) + 1
        if name in LOG.timed:
            import torch
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
    rc = getattr(lib, name)(*args)
    if ev is not None:
        ev[1].record()
        LOG.events.append((name, ev[0], ev[1], nbytes))
    if rc != 0:
        msg = lib.a2d_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 3:
            raise TimeoutError(msg)
        raise KernelError(msg)
