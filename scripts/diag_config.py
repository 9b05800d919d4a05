"""Diagnostic: run one config's pipeline on a query subset with per-phase timings (GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_11076_b200 as t  # noqa: E402

cfg = int(sys.argv[1])
metric = sys.argv[2]
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 8
sh = t.synth_shape(cfg, 0)
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
qs = qs[:nq]
st = t.Store(db)
plan = t.Plan(st, nq, sh["len"], metric, sh["r"], sh["k"])
plan.set_timing(True)
for rep in range(3):
    t0 = time.perf_counter()
    plan.set_queries(qs)
    plan.execute()
    idx, dist, ctr = plan.fetch()
    dt = time.perf_counter() - t0
    s = plan.stats()
    print(f"rep {rep}: wall {dt * 1e3:.2f} ms",
          {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}, flush=True)
print("ctr q0..3", ctr[:4].tolist())
print("idx q0", idx[0].tolist(), "dist", dist[0].tolist())
