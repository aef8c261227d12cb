"""Per-kernel totals of one bench step from an ncu metrics capture ->
profiles/ncu_step_<config>.json (read by bench.py's roofline).

    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file step.csv -k regex:"k_" \
        python bench.py --config c118 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --profile-step
    python tools/ncu_step_metrics.py c118 step.csv [--skip-launches K]

bench.py --profile-step marks the profiled step with a cudaProfilerStart/Stop
range, so the capture (run with --profile-from-start off) holds exactly one
step's launches. Instruction counts (warp-level smsp__inst_executed) are
properties of the workload and kernels, not of the clock: bench.py divides
them by its own CUDA-event stage time to get the achieved issue rate.
"""
import collections
import csv
import json
import re
import sys
from pathlib import Path

OUT_DIR = Path(__file__).resolve().parents[1] / "profiles"
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "": 1}


def short(name):
    return re.sub(r"\(.*$", "", name).replace("void ", "").replace("qvmc_b200::", "").strip()


def main(cfg, path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    idx = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = collections.OrderedDict()
    for r in rows[1:]:
        k = short(r[idx["Kernel Name"]])
        m = r[idx["Metric Name"]]
        v = float(r[idx["Metric Value"]].replace(",", "")) * SCALE.get(r[idx["Metric Unit"]], 1)
        d = per.setdefault(k, {"launch_ids": set(), "time_ms": 0.0, "warp_inst": 0.0, "dram_bytes": 0.0})
        d["launch_ids"].add(r[idx["ID"]])
        if m == "gpu__time_duration.sum":
            d["time_ms"] += v
        elif m == "smsp__inst_executed.sum":
            d["warp_inst"] += v
        elif m.startswith("dram__bytes"):
            d["dram_bytes"] += v
    out = {}
    for k, d in per.items():
        out[k] = {"launches": len(d["launch_ids"]), "time_ms_ncu": d["time_ms"], "warp_inst": d["warp_inst"],
                  "dram_bytes": d["dram_bytes"]}
    tot_t = sum(v["time_ms_ncu"] for v in out.values())
    for v in out.values():
        v["share_of_step_ncu"] = v["time_ms_ncu"] / tot_t if tot_t else 0.0
    res = {"config": cfg, "source": Path(path).name, "kernels": out,
           "note": "one bench step, ncu --clock-control none, serialised and cold-cache per launch"}
    f = OUT_DIR / f"ncu_step_{cfg}.json"
    f.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
