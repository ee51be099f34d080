"""Split an ncu source-page SASS export (--page source --csv --print-source sass)
into address ranges and sum stall samples, instructions, L1 tag requests and
L2 sectors per range -- e.g. pass 1 (block loop) vs pass 2 of a draw kernel.

    python tools/ncu_sass_split.py report.csv [hex_lo-hex_hi ...]
Without ranges it prints every memory instruction with its metrics."""
import csv
import sys


def rows(path):
    with open(path) as fh:
        r = csv.reader(fh)
        next(r)
        hdr = next(r)
        for row in r:
            if len(row) == len(hdr):
                yield dict(zip(hdr, row))


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    path = sys.argv[1]
    data = list(rows(path))
    keys = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Tag Requests Global",
            "L2 Theoretical Sectors Global", "L1 Wavefronts Shared"]
    if len(sys.argv) == 2:
        for d in data:
            if any(t in d["Source"] for t in ("LDG", "STG", "LDS", "STS", "LDL", "STL", "ATOM", "RED")):
                print(d["Address"], d["Source"][:60].ljust(60), *(int(num(d[k])) for k in keys))
        return
    tot = {k: sum(num(d[k]) for d in data) for k in keys}
    print("total", {k.split(" (")[0]: int(v) for k, v in tot.items()})
    for rg in sys.argv[2:]:
        lo, hi = (int(x, 16) for x in rg.split("-"))
        sel = [d for d in data if lo <= int(d["Address"], 16) < hi]
        s = {k: sum(num(d[k]) for d in sel) for k in keys}
        print(rg, {k.split(" (")[0]: f"{int(v)} ({v / max(tot[k], 1):.1%})" for k, v in s.items()})


if __name__ == "__main__":
    main()
