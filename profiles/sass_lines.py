"""Per-source-line instruction counts and stall samples of one kernel from
an ncu capture, by aligning ncu's SASS page with nvdisasm's line table.

    nvcc <build flags> -lineinfo -cubin -o /tmp/harl.cubin csrc/harl_b200.cu
    nvdisasm --print-line-info /tmp/harl.cubin > /tmp/harl_lines.sass
    ncu -i X.ncu-rep --page source --csv --print-source sass > X.sass.csv
    python profiles/sass_lines.py /tmp/harl_lines.sass <mangled-name-prefix> X.sass.csv [N]

(the cubin must come from the same sources and flags as the profiled
library; the script checks the opcode sequence matches)."""

import csv
import re
import sys
from collections import Counter


def main():
    sass, prefix, ncu_csv = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    lines = open(sass).read().split("\n")
    start = [i for i, l in enumerate(lines)
             if "section" in l and ".text." + prefix in l][0]
    insts, cur = [], None
    for l in lines[start + 1:]:
        if ".section" in l and insts:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            insts.append((cur, m.group(2)))
    rows = list(csv.reader(open(ncu_csv)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    data, seen = [], set()
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":   # the next kernel of the capture
            break
        if len(r) <= max(ia, iex, iss) or r[ia] in seen:
            continue
        seen.add(r[ia])
        data.append((int(r[iex] or 0), int(r[iss] or 0), r[isrc]))
    if len(data) != len(insts):
        sys.exit(f"instruction count mismatch: ncu {len(data)} vs "
                 f"cubin {len(insts)} (rebuild the cubin from the profiled "
                 f"sources)")
    ex, st = Counter(), Counter()
    for (cnt, smp, _), (loc, _) in zip(data, insts):
        ex[loc] += cnt
        st[loc] += smp
    tot, ts = sum(ex.values()) or 1, sum(st.values()) or 1
    print(f"warp instructions {tot}, stall samples {ts}")
    for loc, v in ex.most_common(top):
        print(f"{100 * v / tot:5.1f}% exec {100 * st[loc] / ts:5.1f}% stall  "
              f"{loc[0]}:{loc[1]}" if loc else f"{100 * v / tot:5.1f}% ?")


if __name__ == "__main__":
    main()
