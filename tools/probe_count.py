"""Time the candidate search alone (the pairs path's counting pass) against the fused step."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2408_07625_b200 as q  # noqa: E402
from paper_2408_07625_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c118"
H, b = synthetic.make_config(cfg)
for _ in range(2):
    q.surrogate_energy(H, b, want_locals=False)
st = q.last_stats(H)
print("fused: index", st["table_ms"], "rows", st["rows_ms"], "pairs/row", st["pairs"] / st["rows"])
for _ in range(2):
    t0 = time.perf_counter()
    p = q.loop_over_terms(b.vectors, H)
    t1 = time.perf_counter()
st = q.last_stats(H)
print("pairs path: index", st["table_ms"], "count pass", st["rows_ms"], "emit+sort", st["moments_ms"],
      "total wall", t1 - t0, "pairs", len(p.entries))
