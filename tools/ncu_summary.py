"""Summarise ncu captures for profiles/: key raw metrics of each --set full
report, and the per-kernel launch-list table (median duration, DRAM bytes,
GB/s vs the measured HBM peak).

    python tools/ncu_summary.py --report a.ncu-rep [--report b.ncu-rep] [--launches l.csv] \
        [--flops NAME=FLOP ...] > profiles/rNN_ncu_summary.md
"""
import argparse, csv, io, json, os, statistics, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_red.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(hdr, units, r)})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--report", action="append", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--flops", action="append", default=[], help="kernel-substring=algorithmic FLOP per launch")
    a = ap.parse_args()
    flops = {k: float(v) for k, v in (x.split("=") for x in a.flops)}
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    for rep in a.report:
        for r in raw(rep):
            name = r.get("Kernel Name", ("?", ""))[0]
            print(f"## {name[:90]}  ({os.path.basename(rep)}, ncu --set full --clock-control none)")
            for k in KEYS:
                if k in r:
                    print(f"- {k}: {r[k][0]} {r[k][1]}")
            try:
                ms = float(r["gpu__time_duration.sum"][0])
                unit = r["gpu__time_duration.sum"][1]
                ms = ms / 1e3 if unit == "us" else ms
                for sub, f in flops.items():
                    if sub in name:
                        print(f"- algorithmic {f / 1e12:.1f} TFLOP / {ms:.1f} ms = {f / ms / 1e9:.0f} TFLOP/s")
                tr = sum(float(r[k][0]) * (1e9 if r[k][1] == "Gbyte" else 1e6 if r[k][1] == "Mbyte" else 1)
                         for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                print(f"- DRAM traffic {tr / 1e9:.2f} GB per launch")
            except (KeyError, ValueError):
                pass
            print()
    if a.launches:
        text = open(a.launches).read()
        text = text[text.index('"ID"'):]
        rows = list(csv.DictReader(io.StringIO(text)))
        per = {}
        for r in rows:
            key = (r["ID"], r["Kernel Name"])
            per.setdefault(key, {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
        agg = {}
        for (i, name), m in per.items():
            agg.setdefault(name, []).append(m)
        print("| kernel | launches | median ms | DRAM read GB | DRAM write GB | GB/s (DRAM) | frac of %.1f |" % peak)
        print("|---|---|---|---|---|---|---|")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "usecond": 1e-3,
                 "msecond": 1, "nsecond": 1e-6}
        for name, ms in agg.items():
            def med(metric):
                vals = [v * scale.get(u, 1) for v, u in (x[metric] for x in ms if metric in x)]
                return statistics.median(vals) if vals else 0.0
            t = med("gpu__time_duration.sum")
            rd, wr = med("dram__bytes_read.sum") / 1e9, med("dram__bytes_write.sum") / 1e9
            gbs = (rd + wr) / (t * 1e-3) if t else 0
            print(f"| {name[:110]} | {len(ms)} | {t:.3f} | {rd:.3f} | {wr:.3f} | {gbs:.0f} | {gbs / peak:.2f} |")


if __name__ == "__main__":
    main()
