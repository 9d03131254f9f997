"""Small fwd + bwd chunk case for compute-sanitizer (racecheck / synccheck /
memcheck) on the sm_100a kernels: MHA and GQA, causal zig-zag ring step with
the fused merge, d = 128 and d = 64, so every warp role, mbarrier pipeline and
TMEM hand-off runs. Exits non-zero if the results disagree with the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__ as g  # noqa: E402

if __name__ == "__main__":
    g.smoke()
    import numpy as np
    import torch

    from oracle import attn2d_oracle as orc
    from paper_2406_18485_b200 import api
    pos = np.arange(256)
    q, k, v = orc.philox_qkv(3, 4, 2, 256, 64)
    do = np.random.Generator(np.random.Philox(4)).standard_normal(q.shape)
    bf = lambda x: torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).double().numpy()  # noqa: E731
    q, k, v, do = bf(q), bf(k), bf(v), bf(do)
    dq, dk, dv = api.attention_backward(*(api.DenseTensor(x, pos) for x in (q, k, v)), torch.from_numpy(do), True)
    rq, rk, rv = orc.attention_grads(q, k, v, do, pos, pos, True)
    err = max(float(np.abs(a.float().cpu().numpy() - b).max()) for a, b in ((dq, rq), (dk, rk), (dv, rv)))
    print(f"d=64 GQA backward max err {err:.2e}")
    sys.exit(0 if err < 2e-2 * 8 else 1)
