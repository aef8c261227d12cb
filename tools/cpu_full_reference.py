"""One capped full-size run of the UNMODIFIED reference path (SURVEY.md §8d:
"time the largest feasible N_unq plus one capped full run").

    python tools/cpu_full_reference.py --config c118 [--threads N] [--cap-s 3000]

find_coupled_pairs(auto -> trie) -> local_energies -> variational_energy over
the whole 1e6-sample set of the config, all host threads, through
oracle/_ref (the reference sources compiled unchanged). The run happens in a
child process killed at --cap-s; the result (or the cap) is written to
profiles/cpu_full_reference_<config>.json, which bench.py folds into
cpu_baseline_detail.full_size_run. Test/bench infrastructure only.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _run(cfg_name, threads, q):
    import bench
    import oracle
    cfg, cm, batch, gen_s = bench.make_inputs(cfg_name)
    c, x, y, z = cm
    t0 = time.perf_counter()
    R = oracle.RefIndex.from_strings(cfg.n_qubits, c, bench.masks_to_strings(cfg.n_qubits, x, y, z))
    index_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, out5, t3, npairs = R.run_path(batch.vectors, batch.log_amps, batch.phases, batch.log_probs, batch.norm,
                                     batch.log_norm, backend=3, threshold=4096, threads=threads, want_locals=False)
    wall = time.perf_counter() - t0
    q.put({"find_coupled_pairs_s": float(t3[0]), "local_energies_s": float(t3[1]),
           "variational_energy_s": float(t3[2]), "seconds": float(t3.sum()), "wall_s": wall,
           "pairs": int(npairs), "pairs_per_row": npairs / batch.size(), "n_unq": batch.size(),
           "e_var": float(out5[0]), "index_build_s": index_s, "inputs_s": gen_s})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c118")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--cap-s", type=float, default=3000.0)
    a = ap.parse_args()
    q = mp.get_context("fork").Queue()
    p = mp.get_context("fork").Process(target=_run, args=(a.config, a.threads, q))
    t0 = time.perf_counter()
    p.start()
    p.join(a.cap_s)
    res = {"config": a.config, "threads": a.threads, "cap_s": a.cap_s, "host": platform.node(),
           "cpu": platform.processor() or platform.machine(),
           "path": "oracle/_ref: find_coupled_pairs(auto -> trie) -> local_energies -> variational_energy, "
                   "unmodified reference sources, whole sample set"}
    if p.is_alive():
        p.kill()
        res |= {"status": "capped", "elapsed_s": time.perf_counter() - t0}
    else:
        res |= {"status": "ok", **q.get()}
        res["value"] = res["n_unq"] / res["seconds"]
        res["unit"] = "unique-sample local energies/s"
    out = ROOT / "profiles" / f"cpu_full_reference_{a.config}.json"
    out.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
