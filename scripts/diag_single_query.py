"""Diagnostic: single-query plan (the reference's call shape) -- phase times and the LB pass's
HBM throughput (fp32 store bytes / LB time) on one config's store."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_11076_b200 as t  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sh = t.synth_shape(cfg, 0)
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
st = t.Store(db)
plan = t.Plan(st, 1, sh["len"], "dtw", sh["r"], sh["k"])
plan.set_timing(True)
rows = []
for rep in range(8):
    plan.set_queries(qs[rep % len(qs)][None])
    plan.execute()
    plan.fetch()
    rows.append(plan.stats())
ph = {k: float(np.median([r[k] for r in rows[2:]])) for k in rows[0]}
gbs = ph["bound_bytes"] / (ph["ms_bound"] * 1e-3) / 1e9
print(f"config {cfg} single query: total {ph['ms_total']:.3f} ms, LB {ph['ms_bound']:.3f} ms "
      f"({gbs:.0f} GB/s over {ph['bound_bytes'] / 1e6:.0f} MB), DP {ph['ms_dp']:.3f} ms, "
      f"select {ph['ms_select']:.3f}, probe {ph['ms_probe_dp']:.3f}")
