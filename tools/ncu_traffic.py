"""DRAM traffic per launch of profiled kernels -> profiles/ncu_traffic.json (read by bench.py).

usage: python tools/ncu_traffic.py CONFIG [--launches-per-step K] NAME=report.ncu-rep [...]
Each report is one `ncu --set full` capture of one launch; the entry records
dram__bytes_read.sum + dram__bytes_write.sum, the kernel's duration and L2 read
sectors, and how many such launches one bench step makes (row batches).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
SCALE = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9, "Tbyte": 1e12, "TB": 1e12}
TSCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units, vals = rows[0], rows[1], rows[2]
    get = lambda k: (float(vals[names.index(k)].replace(",", "")), units[names.index(k)])
    rd, ru = get("dram__bytes_read.sum")
    wr, wu = get("dram__bytes_write.sum")
    du, dun = get("gpu__time_duration.sum")
    l2, _ = get("lts__t_sectors_srcunit_tex_op_read.sum")
    out = {"kernel": vals[names.index("Kernel Name")], "dram_bytes": rd * SCALE[ru] + wr * SCALE[wu],
           "duration_ms": du * TSCALE[dun], "l2_read_sectors": l2}
    for key, metric in (("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        ("inst_executed", "smsp__inst_executed.sum"),
                        ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                        ("l2_throughput_pct", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed")):
        if metric in names:
            out[key] = get(metric)[0]
    return out


def main(cfg, specs):
    per_step = 1
    if specs and specs[0] == "--launches-per-step":
        per_step, specs = int(specs[1]), specs[2:]
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    entry = data.setdefault(cfg, {})
    for spec in specs:
        name, rep = spec.split("=", 1)
        entry[name] = metrics(rep) | {"report": Path(rep).name, "launches_per_step": per_step}
    OUT.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
