"""Histogram of a kernel's SASS by execution count, from an ncu report's source page:
    python tools/ncu_sass_hist.py report.ncu-rep
Groups the static instructions by their per-instruction warp-level execution count
(blocks of straight-line code share one), largest dynamic share first."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                                  text=True)
    rows = list(csv.reader(io.StringIO(out)))
    k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")   # after the "Kernel Name" line
    rows = rows[k:]
    hdr = rows[0]
    ie = next(i for i, h in enumerate(hdr) if h.strip() == "Instructions Executed")
    src = next(i for i, h in enumerate(hdr) if h.strip() == "Source")
    samp = next((i for i, h in enumerate(hdr) if h.strip() == "Warp Stall Sampling (All Samples)"), None)
    groups = defaultdict(lambda: [0, 0.0, []])
    total, tots = 0, 0.0
    for r in rows[1:]:
        try:
            n = int(float(r[ie].replace(",", "") or 0))
        except ValueError:
            continue
        s = float(r[samp].replace(",", "") or 0) if samp is not None else 0.0
        total += n
        tots += s
        if n:
            g = groups[n]
            g[0] += 1
            g[1] += s
            g[2].append(r[src].strip())
    print(f"total dynamic warp instructions: {total}")
    for n, (k, s, ins) in sorted(groups.items(), key=lambda t: -t[0] * t[1][0])[:12]:
        print(f"exec count {n:10d}: {k:4d} static instr, {100 * n * k / total:5.1f}% of dynamic instr, "
              f"{100 * s / max(tots, 1):5.1f}% samples")


if __name__ == "__main__":
    main()
