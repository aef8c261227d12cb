"""Aggregate an ncu --page source --print-source sass,cuda CSV by CUDA source line.

usage: ncu -i rep --page source --csv --print-source sass,cuda > x.csv; python tools/ncu_lines.py x.csv [N]
"""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    cur = None
    agg = collections.defaultdict(lambda: [0, 0, ""])

    def num(v):
        try:
            return int(v)
        except ValueError:
            return 0

    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        if len(r) > 8 and r[0] not in ("", "Line No"):  # per-line aggregate rows
            k = (cur, int(r[0]))
            agg[k][0] += num(r[4])
            agg[k][1] += num(r[7])
            agg[k][2] = r[1]
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"{'file':18} {'line':>5} {'stall%':>6} {'inst%':>6}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0][:18]:18} {k[1]:>5} {100 * v[0] / ts:6.1f} {100 * v[1] / ti:6.1f} | {v[2][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
