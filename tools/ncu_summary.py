"""Summarise ncu reports into markdown (run here, on the copied .ncu-rep files).

    python tools/ncu_summary.py gpurun_out/prof_rows_k1024.ncu-rep [...] > profiles/xxx.md
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.per_cycle_active", "active warps/SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def summarise(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"### `{path.split('/')[-1]}`\n"]
    for d in rows[2:]:
        name = d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"**{name[:110]}**\n")
        out.append("| metric | value |\n|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"| {label} (`{m}`) | {d[i]} {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
                try:
                    stalls.append((float(d[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{h} {v / tot * 100:.0f}%" for v, h in sorted(stalls, reverse=True)[:4])
        out.append(f"| top stall reasons (pc sampling) | {top} |\n")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
