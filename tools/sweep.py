"""Factorization sweep (BASELINE config 5 style): every (d_hp, d_cp, w,
placement) valid for the given GPU counts, one bench.py run each.

    python tools/sweep.py --gpus 2 4 --seq 524288 --out profiles/sweep.jsonl
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_18485_b200.config import (ClusterConfig, ModelConfig, ParallelConfig,  # noqa: E402
                                          Placement, validate)


def configs(n, model):
    for d_hp in range(1, n + 1):
        if n % d_hp:
            continue
        d_cp = n // d_hp
        for w in range(1, d_cp + 1):
            if d_cp % w:
                continue
            for pl in Placement:
                par = ParallelConfig(d_hp=d_hp, d_cp=d_cp, inner_ring=w, placement=pl)
                if validate(model, par, ClusterConfig()).ok:
                    yield d_hp, d_cp, w, pl.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--seq", type=int, default=524288)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    ap.add_argument("--timeout", type=int, default=600)
    ap.add_argument("--placements", nargs="+", default=["head_first", "context_first"])
    ap.add_argument("--bench-args", default="", help="extra bench.py arguments, e.g. '--no-check'")
    a = ap.parse_args()
    model = ModelConfig(seq_len=a.seq, heads=a.heads, kv_heads=a.kv_heads, hidden=a.heads * 128)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    port = 29700
    with open(a.out, "a") as f:
        for n in a.gpus:
            for d_hp, d_cp, w, pl in configs(n, model):
                if pl not in a.placements:
                    continue
                port += 1
                cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                       "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
                       "--gpus", str(n), "--steps", str(a.steps), "--warmup", str(a.warmup), "--seq", str(a.seq),
                       "--heads", str(a.heads), "--kv-heads", str(a.kv_heads), "--d-hp", str(d_hp),
                       "--d-cp", str(d_cp), "--w", str(w), "--placement", pl, "--no-e2e", "--no-cpu",
                       *a.bench_args.split()]
                try:
                    r = subprocess.run(cmd, capture_output=True, text=True, timeout=a.timeout, cwd=ROOT)
                    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
                    rec = json.loads(line[-1]) if line else {"error": r.stderr[-1500:]}
                except subprocess.TimeoutExpired:
                    rec = {"error": "timeout"}
                rec["sweep"] = {"n": n, "d_hp": d_hp, "d_cp": d_cp, "w": w, "placement": pl, "seq": a.seq}
                f.write(json.dumps(rec) + "\n")
                f.flush()
                short = {k: rec.get(k) for k in ("value", "tflops_per_gpu", "ms_per_step")}
                ex = (rec.get("exposed_comm") or {}).get("frac")
                print(json.dumps({**rec["sweep"], **short, "exposed": ex, "err": rec.get("error", "")[:200]}),
                      flush=True)


if __name__ == "__main__":
    main()
