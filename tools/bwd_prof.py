"""Where does each warp role of fa_bwd_kernel wait? Runs one backward at the
bench shape through the instrumented library (build.py --profile:
-DA2D_PROFILE) and prints, per role, the fraction of its cycles spent blocked
on each barrier (clock64 around every mbarrier wait, summed over CTAs).

    python -m paper_2406_18485_b200.build --profile
    python tools/bwd_prof.py [--seq 131072] [--heads 32] [--kv-heads 32] [--dim 128]
"""

import argparse
import ctypes
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["A2D_LIB"] = os.path.join(ROOT, "paper_2406_18485_b200", "lib",
                                     "libattn2d_sm100_prof%s.so" % (("_" + os.environ["A2D_PROF_VARIANT"].lower())
                                                                   if os.environ.get("A2D_PROF_VARIANT") else ""))

import torch  # noqa: E402

from paper_2406_18485_b200 import _lib  # noqa: E402
from paper_2406_18485_b200 import kernels as K  # noqa: E402

SLOTS = {
    "mma": ["kv_full", "qdo_full(TMA)", "ds_full(softmax)", "dq_empty(drain)", "-", "-", "-", "total"],
    "pds": ["qdo_full(stats)", "s_full(MMA S,dP)", "ds_free(dQ GEMM read dS)", "-", "-", "-", "-", "total"],
    "drain": ["dq_full(dQ GEMM)", "bulk_wait_read(TMA reduce)", "-", "-", "-", "-", "-", "total"],
    "tma": ["qdo_empty(MMA frees stage)", "-", "-", "-", "-", "-", "-", "total"],
}
# the 128-query kernel (fa_bwd_q128.cuh, the D = 128 default; A2D_BWD_VARIANT=6 selects the one above)
SLOTS_Q128 = {
    "mma": ["kv_full", "qdo_full(TMA)", "p_full(softmax P)", "dq_empty(drain TMEM read)", "dst_full(softmax dS TMEM)",
            "dss_full(softmax dS smem)", "do_full(TMA dO)", "total"],
    "pds": ["qdo_full(stats)", "s_full(MMA S)", "dp_full(MMA dP)", "dsbuf_free(drain staging)", "-", "-", "-", "total"],
    "drain": ["dq_full(dQ GEMM)", "bulk_wait_read(box b-2)", "-", "-", "-", "-", "-", "total"],
    "tma": ["q_empty(dK frees Q)", "do_empty(dV frees dO)", "-", "-", "-", "-", "-", "total"],
}
FWD_SLOTS = {
    "mma": ["v_full(TMA)", "p_full0(softmax WG0)", "k_full(TMA)", "p_full1(softmax WG1)", "-", "-", "-", "total"],
    "softmax0": ["s_full(MMA QK)", "-", "-", "-", "-", "-", "-", "total"],
    "softmax1": ["s_full(MMA QK)", "-", "-", "-", "-", "-", "-", "total"],
    "tma": ["k_empty", "v_empty", "-", "-", "-", "-", "-", "total"],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--pass", dest="which", default="bwd", choices=["bwd", "fwd"])
    a = ap.parse_args()
    lib = _lib.load(os.environ["A2D_LIB"])
    lib.a2d_prof_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.a2d_prof_read_fwd.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.a2d_prof_ablate(int(os.environ.get("A2D_ABLATE", "0")))
    dev = torch.device("cuda:0")
    H, Hkv, S, d = a.heads, a.kv_heads, a.seq, a.dim
    g = torch.Generator(device=dev).manual_seed(0)
    q, do = (torch.randn((H, S, d), device=dev, generator=g).to(torch.bfloat16) for _ in range(2))
    k, v = (torch.randn((Hkv, S, d), device=dev, generator=g).to(torch.bfloat16) for _ in range(2))
    plan = K.ChunkPlan(torch.arange(S, dtype=torch.int32, device=dev))
    scale = 1 / math.sqrt(d)
    lse = torch.empty((H, S), dtype=torch.float32, device=dev)
    out = torch.empty_like(q)
    K.fwd_chunk(q, k, v, plan, plan, True, scale, lse, None, out)
    lse2, delta = K.bwd_preprocess(out, do, lse)
    dq_acc = K.dq_acc_t(H, S, dev, d)
    dk = torch.empty((Hkv, S, d), dtype=torch.float32, device=dev)
    dv = torch.empty_like(dk)
    buf = (ctypes.c_ulonglong * 32)()
    if a.which == "fwd":
        torch.cuda.synchronize()
        lib.a2d_prof_read_fwd(buf, 32)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.fwd_chunk(q, k, v, plan, plan, True, scale, lse, None, out)
        e1.record()
        torch.cuda.synchronize()
        lib.a2d_prof_read_fwd(buf, 32)
        ms = e0.elapsed_time(e1)
        res = {"shape": vars(a), "fwd_ms": ms, "fwd_tflops": 2.0 * S * S * H * d / ms / 1e9}
        for role, base in (("mma", 0), ("softmax0", 8), ("softmax1", 16), ("tma", 24)):
            vals = list(buf[base:base + 8])
            tot = vals[7] or 1
            res[role] = {FWD_SLOTS[role][i]: round(vals[i] / tot, 4) for i in range(7) if FWD_SLOTS[role][i] != "-"}
            res[role]["total_Gcycles"] = vals[7] / 1e9
        print(json.dumps(res, indent=1))
        return
    K.bwd_chunk(q, k, v, do, plan, plan, lse2, delta, dq_acc, dk, dv, False, True, scale)  # warm-up
    torch.cuda.synchronize()
    lib.a2d_prof_read(buf, 32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K.bwd_chunk(q, k, v, do, plan, plan, lse2, delta, dq_acc, dk, dv, False, True, scale)
    e1.record()
    torch.cuda.synchronize()
    lib.a2d_prof_read(buf, 32)
    ms = e0.elapsed_time(e1)
    res = {"shape": vars(a), "bwd_ms": ms, "bwd_tflops": 2.5 * 2.0 * S * S * H * d / ms / 1e9}
    slots = SLOTS_Q128 if d == 128 and os.environ.get("A2D_BWD_VARIANT", "0") in ("0", "7", "8", "9", "10", "11", "13") else SLOTS
    for role, base in (("mma", 0), ("pds", 8), ("drain", 16), ("tma", 24)):
        vals = list(buf[base:base + 8])
        tot = vals[7] or 1
        res[role] = {slots[role][i]: round(vals[i] / tot, 4) for i in range(7) if slots[role][i] != "-"}
        res[role]["total_Gcycles"] = vals[7] / 1e9
    if os.environ.get("A2D_TRACE"):
        tb = (ctypes.c_longlong * 512)()
        lib.a2d_prof_trace(tb)
        names = ["mma:dV(i)", "mma:S(i+1)", "mma:dK(i)", "mma:dQ(i)", "mma:dq_empty", "mma:dP(i+1)",
                 "sm:s_full", "sm:P_done", "sm:dp_full", "sm:dS_done", "sm:sts_start", "sm:sts_done",
                 "sm1:P_done", "dr:dq_full", "dr:dq_empty", "dr:end"]
        t0 = tb[0]
        res["trace_cycles_rel_to_first_dV"] = {n: [tb[i * 16 + k] - t0 for i in range(32)] for k, n in enumerate(names)}
        per = [(tb[(i + 1) * 16] - tb[i * 16]) for i in range(31)]
        res["trace_period"] = per
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
