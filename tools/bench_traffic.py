"""Refresh profiles/ncu_summary.json's `bfly_lda_k1024` entry (the numbers
behind bench.py's roofline.traffic and roofline.hbm) from an ncu launch list
of the bench's own draw:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none \
        -k "regex:bfly_kernel|lda_" --csv --log-file launches.csv \
        python bench.py --steps 2 --warmup 1 --no-cpu --no-dropin --no-e2e --no-sampler

    python tools/bench_traffic.py launches.csv HEAD [--launches-per-draw 4]

The first draw (warm-up, cold L2) is excluded; the rest are averaged per draw.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("head")
    ap.add_argument("--launches-per-draw", type=int, default=4)
    ap.add_argument("--copy-to", default=None, help="also copy the csv here (profiles/...)")
    args = ap.parse_args()
    rows = [r for r in csv.reader(open(args.csv)) if len(r) > 10]
    hdr = rows[0]
    iid, iname, imet, ival = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[int(r[iid])][r[imet]] = float(r[ival].replace(",", ""))
        names[int(r[iid])] = r[iname]
    ids = sorted(per)
    L = args.launches_per_draw
    if len(ids) < 2 * L:
        raise SystemExit(f"need at least two draws of {L} launches, got {len(ids)} launches")
    kept = ids[L:]  # drop the warm-up draw
    draws = len(kept) / L
    tot = lambda m: sum(per[i].get(m, 0.0) for i in kept)  # noqa: E731
    rd, wr = tot("dram__bytes_read.sum"), tot("dram__bytes_write.sum")
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(path))
    src_csv = args.copy_to or args.csv
    summ["bfly_lda_k1024"] = {
        "kernel": names[kept[0]].split("(")[0] + " (the bench's LDA draw, vocabulary-tiled, run-padded, "
                  f"{L} launches per draw)",
        "source": f"{src_csv} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                  "lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none "
                  "-k regex:bfly_kernel|lda_ python bench.py --steps 2 --warmup 1 ...); the first draw (warm-up) "
                  "excluded",
        "head": args.head,
        "launches_per_draw": L,
        "draws_captured": draws,
        "dram_bytes_per_draw": (rd + wr) / draws,
        "dram_read_bytes_per_draw": rd / draws,
        "dram_write_bytes_per_draw": wr / draws,
        "lts_bytes_per_draw": tot("lts__t_bytes.sum") / draws,
        "ncu_ms_per_draw": tot("gpu__time_duration.sum") / 1e6 / draws,
        "lts_tex_read_bytes_per_draw": tot("lts__t_sectors_srcunit_tex_op_read.sum") * 32 / draws,
    }
    if args.copy_to and os.path.abspath(args.csv) != os.path.join(ROOT, args.copy_to):
        import shutil

        shutil.copyfile(args.csv, os.path.join(ROOT, args.copy_to))
    with open(path, "w") as f:
        json.dump(summ, f, indent=1)
        f.write("\n")
    print(json.dumps(summ["bfly_lda_k1024"], indent=1))


if __name__ == "__main__":
    main()
