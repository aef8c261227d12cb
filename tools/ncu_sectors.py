"""L2 sectors requested per CUDA source line from an ncu --page source CSV (sass,cuda).

usage: ncu -i rep --page source --csv --print-source sass,cuda > x.csv; python tools/ncu_sectors.py x.csv [N]
"""
import collections
import csv
import sys


def main(path, top=25):
    cur, hdr = None, None
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    for r in csv.reader(open(path)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            d = dict(zip(hdr, r))
            try:
                sec = float(d.get("L2 Theoretical Sectors Global", "0") or 0)
                st = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            except ValueError:
                continue
            k = (cur, int(r[0]))
            agg[k][0] += sec
            agg[k][1] += st
            agg[k][2] = r[1]
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"total L2 sectors requested: {tot:.4g} ({tot * 32 / 1e9:.2f} GB)")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0][:18]:18} {k[1]:>5} {100 * v[0] / tot:6.1f}% {v[0] * 32 / 1e9:8.2f} GB | {v[2][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
