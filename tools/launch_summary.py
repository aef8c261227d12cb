"""Per-kernel totals from an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python tools/launch_summary.py launches.csv > profiles/<round>_launches.txt
The list is cold-cache and serialised: compare each kernel's SHARE of a step,
not the absolute times, with bench.py's CUDA-event numbers.
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name)
    return name.replace("void ", "").replace("qvmc_b200::", "")[:80]


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    recs = [dict(zip(hdr, r)) for r in rows[1:] if r[hdr.index("Metric Name")] == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    for d in recs:
        k = short(d["Kernel Name"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"# {len(recs)} launches, {tot / 1e3:.2f} ms total device time (ncu, cold cache, serialised)")
    print(f"{'kernel':80} {'launches':>8} {'total us':>12} {'share':>7}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:80} {n:>8} {us:>12.1f} {100 * us / tot:>6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
