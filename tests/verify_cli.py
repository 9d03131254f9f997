"""Parity CLI for the B200 2D-Attention path — mirrors the reference's
``attn2d verify`` (``/root/reference/pkg/src/attn2d/cli.py:46-122``).

    python tests/verify_cli.py [--seq S] [--dsp N] [--smax 256] [--seed 0]
                               [--precision f64|f32] [--inject-fault]

Runs ``paper_2406_18485_b200.api.run_2d_attention`` (the B200 kernels, global
view on one GPU) over the reference's lattice — H=4, hidden=32, H_kv in
{2, 4}, S in {32, 64}, d_sp in {1, 2, 4, 8}, d_hp in {1, 2, 4}, every inner
ring w | d_cp, both placements, causal and not — and compares every output
with the f64 oracle's full attention (test infrastructure, used only as the
checker). Same exit codes as the reference: 0 all within tolerance, 1 a
configuration failed (``--inject-fault`` negates the first output to prove
detection, cli.py:93-95), 2 configuration error.

Tolerance: the reference compares its own numpy path at 1e-10 (f64) / 1e-5
(f32); the B200 kernels compute in bf16 with fp32 accumulation, so the bar is
the north star's max-abs 2e-2 for both precisions (inputs are rounded to
bf16 first; the oracle sees the same rounded values).
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EXIT_OK, EXIT_FAIL, EXIT_CONFIG = 0, 1, 2
TOLERANCE = 2e-2


def _rng(seed: int):
    return np.random.Generator(np.random.Philox(seed))


def _divisors(n: int):
    return [x for x in range(1, n + 1) if n % x == 0]


def _lattice(args):
    """(heads, kv_heads, S, d, seed) x causal x (d_hp, d_cp, w, placement).
    Default: the `attn2d verify` lattice (cli.py:58-91, 304 configurations);
    --acceptance: test_acceptance.py criterion 1's (:53-91, > 500)."""
    from paper_2406_18485_b200.config import Placement
    if args.acceptance:
        problems = [(h, kv, s, 8, 1000 + h + kv + s) for h in (4, 8) for kv in sorted({2, 4, h})
                    for s in (16, 32, 64)]
        sps, hps = (1, 2, 4, 8, 16), None
    else:
        seqs = (args.seq,) if args.seq else (32, 64)
        problems = [(4, kv, s, 8, None) for kv in (2, 4) for s in seqs if s <= args.smax]
        sps, hps = ((args.dsp,) if args.dsp else (1, 2, 4, 8)), (1, 2, 4)
    for heads, kv, S, d, seed in problems:
        for causal in (False, True):
            grids = []
            for d_sp in sps:
                if S % (2 * d_sp):
                    continue
                for d_hp in (hps or _divisors(d_sp)):
                    if d_sp % d_hp or d_hp > heads or heads % d_hp:
                        continue
                    d_cp = d_sp // d_hp
                    for w in (x for x in (1, 2, 4, 8, 16) if d_cp % x == 0 and x <= d_cp):
                        for pl in Placement:
                            grids.append((d_hp, d_cp, w, pl))
            yield (heads, kv, S, d, seed, causal, grids)


def verify(args) -> int:
    import torch

    from oracle import attn2d_oracle as orc
    from paper_2406_18485_b200 import api
    from paper_2406_18485_b200.config import ClusterConfig, ModelConfig, ParallelConfig

    if args.smax > 256:
        print("error: verify is desk-scale only (S <= 256)", file=sys.stderr)
        return EXIT_CONFIG
    if args.dsp is not None and args.seq is not None and args.seq % (2 * args.dsp) != 0:
        print(f"error: S={args.seq} not divisible by 2*d_sp={2 * args.dsp}", file=sys.stderr)
        return EXIT_CONFIG
    dtype = np.float64 if args.precision == "f64" else np.float32
    cluster = ClusterConfig()
    rng = _rng(args.seed)
    worst, failures, first, n = 0.0, [], True, 0
    for heads, kv_heads, seq_len, d, seed, causal, grids in _lattice(args):
        model = ModelConfig(seq_len=seq_len, heads=heads, kv_heads=kv_heads, hidden=heads * d)
        g = _rng(seed) if seed is not None else rng
        vals = [g.standard_normal((h, seq_len, d)).astype(dtype) for h in (heads, kv_heads, kv_heads)]
        vals = [torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).double().numpy() for x in vals]
        pos = np.arange(seq_len)
        ref, _ = orc.attention(*vals, pos, pos, causal)
        q, k, v = (api.DenseTensor(x, pos) for x in vals)
        for d_hp, d_cp, w, placement in grids:
            par = ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=w, placement=placement)
            try:
                out = api.run_2d_attention(q, k, v, model, par, cluster, causal)
            except ValueError as e:  # the reference raises for the same configs
                print(f"error: {e}", file=sys.stderr)
                return EXIT_CONFIG
            got = out.values.float().cpu().double().numpy()
            if args.inject_fault and first:
                got = -got
                first = False
            delta = float(np.max(np.abs(got - ref)))
            worst = max(worst, delta)
            n += 1
            name = (f"H={heads} H_kv={kv_heads} S={seq_len} causal={causal} d_hp={d_hp} "
                    f"d_cp={d_cp} w={w} {placement.value}")
            print(f"{name}: max|delta|={delta:.3e}")
            if delta > TOLERANCE:
                failures.append(name)
    if failures:
        print(f"FAIL: {len(failures)} configuration(s) exceed {TOLERANCE:g}:")
        for name in failures:
            print(f"  {name}")
        return EXIT_FAIL
    print(f"OK: all {n} configurations within {TOLERANCE:g} (worst {worst:.3e})")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="verify", description=__doc__.split("\n\n")[0])
    ap.add_argument("--seq", type=int, default=None)
    ap.add_argument("--dsp", type=int, default=None)
    ap.add_argument("--smax", type=int, default=256)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--precision", choices=["f64", "f32"], default="f64")
    ap.add_argument("--inject-fault", action="store_true")
    ap.add_argument("--acceptance", action="store_true",
                    help="the larger lattice of the reference's acceptance criterion 1 (test_acceptance.py:53-91)")
    return verify(ap.parse_args(argv))


if __name__ == "__main__":
    sys.exit(main())
