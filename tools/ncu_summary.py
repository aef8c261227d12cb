"""Text summary of an ncu report for profiles/: key section metrics + hottest source lines.

usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Registers Per Thread", "Grid Size", "Block Size",
        "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Static Shared Memory Per Block"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    print(f"# ncu summary of {rep.split('/')[-1]}")
    kern = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if kern is None:
            kern = d.get("Kernel Name")
            print(f"kernel: {kern}\n")
        if d.get("Metric Name") in KEEP:
            print(f"{d['Section Name']:<34} {d['Metric Name']:<40} {d['Metric Value']:>16} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        names, units, vals = raw[0], raw[1], raw[2]
        print()
        for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
                     "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            if want in names:
                i = names.index(want)
                print(f"{want:<64} {vals[i]:>16} {units[i]}")
    print("\n## hottest source lines (warp-stall samples / executed instructions)\n")
    sys.stdout.flush()
    src = run([rep, "--page", "source", "--csv", "--print-source", "sass,cuda"])
    import collections
    agg = collections.defaultdict(lambda: [0, 0, ""])
    cur = None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        if len(r) > 8 and r[0] not in ("", "Line No"):
            try:
                agg[(cur, int(r[0]))][0] += int(r[4] or 0)
                agg[(cur, int(r[0]))][1] += int(r[7] or 0)
            except ValueError:
                pass
            agg[(cur, int(r[0]))][2] = r[1]
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"{k[0][:20]:20} {k[1]:>5} stall {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}% | {v[2][:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
