"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total/avg device time and share."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = (h.index("Kernel Name"), h.index("Metric Value"),
                  h.index("Metric Unit"))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
             "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if name.endswith("k_spin"):
            continue   # bench's per-kernel timer (untimed profiled episode)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(v for _, v in agg.values())
    out = ["| kernel | launches | total us | avg us | share |",
           "|---|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k[:70]} | {c} | {v:.1f} | {v / c:.1f} | {v / tot:.3f} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
