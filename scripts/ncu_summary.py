"""Summarise ncu outputs into profiles/ (run here, on the CPU box, after gpurun).

    python scripts/ncu_summary.py --rep gpurun_out/prof_full.ncu-rep --out profiles/r01_ncu_full.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/r01_launches.md
    python scripts/ncu_summary.py --rep ... --traffic-json profiles/traffic.json

The launch list (gpu__time_duration per launch) is cold-cache and serialised: read the
per-kernel SHARE of the step from it, not absolute times.
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc_pipe_active_%"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_mem_active_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def _to_bytes(v, unit):
    f = float(v.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return f * mult


def summarize_rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        rec = {"kernel": r[h.index("Kernel Name")]}
        for k, short in KEYS:
            if k in h:
                i = h.index(k)
                rec[short] = f"{r[i]} {units[i]}".strip()
                if k.startswith("dram__bytes"):
                    rec[short + "_bytes"] = _to_bytes(r[i], units[i])
        out.append(rec)
    return out


def summarize_launches(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if "Kernel Name" in l)
    rows = list(csv.reader(txt[start:]))
    h, data = rows[0], rows[1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        name = re.sub(r"\(.*", "", r[ki])[:70]
        agg.setdefault(name, []).append(v)
    total = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
             "share": sum(v) / total} for k, v in agg.items()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    lines = [f"# {a.title or a.out}", ""]
    if a.rep:
        recs = summarize_rep(a.rep)
        lines.append(f"ncu --set full capture: `{a.rep}` ({len(recs)} launches)")
        lines.append("")
        cols = ["kernel"] + [s for _, s in KEYS]
        lines.append("| " + " | ".join(cols) + " |")
        lines.append("|" + "---|" * len(cols))
        for r in recs:
            lines.append("| " + " | ".join(str(r.get(c, ""))[:48] for c in cols) + " |")
        if a.traffic_json:
            tj = {}
            for r in recs:
                k = r["kernel"]
                tj.setdefault(k, []).append(r.get("dram_read_bytes", 0) + r.get("dram_write_bytes", 0))
            json.dump({k: sum(v) / len(v) for k, v in tj.items()}, open(a.traffic_json, "w"), indent=1)
    if a.launches:
        recs = summarize_launches(a.launches)
        lines.append(f"ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised):"
                     f" `{a.launches}`")
        lines.append("")
        lines.append("| kernel | launches | mean us | total us | share |")
        lines.append("|---|---|---|---|---|")
        for r in recs:
            lines.append(f"| {r['kernel']} | {r['launches']} | {r['mean_us']:.1f} | {r['total_us']:.1f} | "
                         f"{100 * r['share']:.1f}% |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
