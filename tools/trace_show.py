"""Print the per-iteration event timeline recorded by the profile build
(A2D_TRACE=1 tools/bwd_prof.py > file.json): cycles relative to each
iteration's dV issue, for a few steady-state iterations."""
import json, sys
for fn in sys.argv[1:]:
    d = json.load(open(fn))
    tr = d["trace_cycles_rel_to_first_dV"]; per = d["trace_period"]
    print(fn, "tflops", round(d["bwd_tflops"]), "period median", sorted(per)[len(per) // 2])
    for i in range(10, 13):
        base = tr["mma:dV(i)"][i]
        print(i, " ".join(f"{n.split(':')[1]}={tr[n][i] - base}" for n in tr))
