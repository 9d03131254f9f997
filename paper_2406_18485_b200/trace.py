"""Measured Chrome traces of one 2D-attention step.

Same output format as the reference simulator's ``export_trace`` (ref
timeline.py:203-219: Chrome Trace Event "X" complete events, microseconds,
``tid`` = rank, ``args.resource``), but the events are MEASURED: the CUDA
events ``dist.Attn2D`` records on the compute stream at every phase boundary
(``record_times``). The planner's prediction for the same configuration
(``planner.predict``) is emitted next to it as pid 1, so the B200 cost model
can be checked against the measurement phase by phase.
"""

from __future__ import annotations

import json

from .config import ModelConfig, ParallelConfig
from .planner import predict

MEASURED_PID, PREDICTED_PID = 0, 1


def _kind(name: str) -> tuple[str, str]:
    """(event kind, resource) of the interval that ENDS at mark `name`."""
    if "a2a" in name:
        return "AlltoAll", "hp_group"
    if ".step" in name:
        return "Compute", "sm"           # ring step: attention kernel (+ hop waits, K4 add)
    return "Compute", "sm"


def phases_from_marks(marks: list[tuple[str, float]]) -> list[tuple[str, float, float]]:
    """[(mark, t_ms)] in record order -> [(phase, start_ms, end_ms)]; a phase is
    named by the mark that closes it ("fwd.start"/"bwd.start" open a pass)."""
    out = []
    for (n0, t0), (n1, t1) in zip(marks, marks[1:]):
        if n1.endswith(".start"):
            continue  # gap between the forward and the backward pass
        out.append((n1, t0, t1))
    return out


def chrome_events(per_rank: dict[int, list[tuple[str, float]]], pid: int = MEASURED_PID) -> list[dict]:
    """Chrome "X" records (µs) from per-rank mark lists (times in ms)."""
    recs = []
    for rank in sorted(per_rank):
        for name, t0, t1 in phases_from_marks(per_rank[rank]):
            kind, res = _kind(name)
            recs.append({"ph": "X", "name": f"{kind} {name}", "ts": t0 * 1e3, "dur": max(0.0, t1 - t0) * 1e3,
                         "pid": pid, "tid": rank, "args": {"resource": res}})
    return recs


def predicted_marks(model: ModelConfig, par: ParallelConfig, causal: bool = True) -> list[tuple[str, float]]:
    """The planner's step model laid out as the same marks (ms) as one rank records."""
    p = predict(model, par, causal=causal)
    d_cp = par.d_cp
    ph = p["t_phases"]
    exposed = p["t_ring_exposed"]
    hop = exposed / 2 / max(1, d_cp - 1) if d_cp > 1 else 0.0
    t, marks = 0.0, [("fwd.start", 0.0)]
    t += ph["fwd.a2a_in"]
    marks.append(("fwd.a2a_in", t))
    for s in range(d_cp):
        t += p["t_fwd"] / d_cp + (hop if s else 0.0)
        marks.append((f"fwd.step{s}", t))
    t += ph["fwd.a2a_out"]
    marks.append(("fwd.a2a_out", t))
    marks.append(("bwd.start", t))
    t += ph["bwd.a2a_in"]
    marks.append(("bwd.a2a_in", t))
    for s in range(d_cp):
        t += p["t_bwd"] / d_cp + (hop if s else 0.0)
        marks.append((f"bwd.step{s}", t))
    marks.append(("bwd.ring", t))
    t += ph["bwd.a2a_out"]
    marks.append(("bwd.a2a_out", t))
    return [(n, x * 1e3) for n, x in marks]


def phase_summary(per_rank: dict[int, list[tuple[str, float]]]) -> dict[str, float]:
    """Max over ranks of the time (ms) spent per phase group."""
    groups: dict[str, float] = {}
    for rank, marks in per_rank.items():
        acc: dict[str, float] = {}
        for name, t0, t1 in phases_from_marks(marks):
            g = name.split(".")[0] + "." + ("ring" if ".step" in name or name.endswith(".ring") else name.split(".")[1])
            acc[g] = acc.get(g, 0.0) + (t1 - t0)
        for g, v in acc.items():
            groups[g] = max(groups.get(g, 0.0), v)
    return groups


def export(path: str, measured: dict[int, list[tuple[str, float]]], model: ModelConfig | None = None,
           par: ParallelConfig | None = None, causal: bool = True) -> dict:
    """Write the trace (measured pid 0 [+ predicted pid 1]) and return a summary."""
    recs = chrome_events(measured, MEASURED_PID)
    summary = {"measured_ms": phase_summary(measured)}
    if model is not None and par is not None:
        pm = predicted_marks(model, par, causal)
        recs += chrome_events({r: pm for r in measured}, PREDICTED_PID)
        summary["predicted_ms"] = phase_summary({0: pm})
    recs.sort(key=lambda r: (r["pid"], r["tid"], r["ts"]))
    with open(path, "w") as f:
        json.dump(recs, f, indent=1, sort_keys=True)
        f.write("\n")
    return summary
