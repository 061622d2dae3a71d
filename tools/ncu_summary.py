"""Summarise an ncu --set full report (raw page) into the metrics DESIGN.md cites.
    python tools/ncu_summary.py report.ncu-rep [label]"""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum"]


def main():
    rep = sys.argv[1]
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for vals in rows[2:]:
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                lines.append(f"{w:58s} {vals[i][:90]:>20s} {units[i]}")
        st = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled")
              and not h.endswith("not_issued")]

        def f(x):
            try:
                return float(x.replace(",", ""))
            except ValueError:
                return 0.0
        tot = sum(f(v) for _, v in st) or 1.0
        lines.append("top warp stall reasons (pc sampling, share of samples):")
        for h, v in sorted(st, key=lambda t: -f(t[1]))[:8]:
            lines.append(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * f(v) / tot:5.1f}%")
        lines.append("")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
