"""Summarise ncu --set full captures (raw page CSV) into a markdown table
and a per-kernel DRAM-traffic json.

    ncu -i X.ncu-rep --page raw --csv > X.raw.csv
    python profiles/ncu_summary.py OUT.md [--traffic OUT.json] X.raw.csv ...

Columns: duration, tensor pipe (cycles active, % of peak elapsed, and the
realtime variant), tensor-core instructions issued, TMEM pipe instructions,
XU (MUFU) pipe, issue activity, warps active, DRAM read/write per launch.
"""

import csv
import json
import re
import sys

COLS = [
    ("time us", "gpu__time_duration.sum"),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe realtime %", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tc inst % active", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"),
    ("tmem inst % active", "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"),
    ("xu (MUFU) % active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("DRAM read MB", "dram__bytes_read.sum"),
    ("DRAM write MB", "dram__bytes_write.sum"),
]
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "s": 1e6, "usecond": 1.0,
         "msecond": 1e3, "nsecond": 1e-3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).strip()}
        d["kernel"] = re.sub(r"^void ", "", d["kernel"])
        for label, m in COLS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = float("nan")
                d[label] = v * SCALE.get(units[i], 1.0)
        out.append(d)
    return out


def main():
    args = sys.argv[1:]
    out_md = args.pop(0)
    traffic = None
    if args and args[0] == "--traffic":
        args.pop(0)
        traffic = args.pop(0)
    lines = []
    tr = {}
    for path in args:
        lines.append(f"\n### {path}\n")
        lines.append("| kernel | " + " | ".join(c for c, _ in COLS) + " |")
        lines.append("|---" * (len(COLS) + 1) + "|")
        for d in load(path):
            lines.append(f"| {d['kernel']} | " + " | ".join(
                f"{d.get(c, float('nan')):.3g}" for c, _ in COLS) + " |")
            t = tr.setdefault(re.sub(r"<.*", "", d["kernel"]), [])
            t.append(1e6 * (d.get("DRAM read MB", 0) + d.get("DRAM write MB", 0)))
    open(out_md, "a").write("\n".join(lines) + "\n")
    if traffic:
        json.dump({k: {"dram_bytes_per_launch": sum(v) / len(v),
                       "launches_captured": len(v)} for k, v in tr.items()},
                  open(traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
