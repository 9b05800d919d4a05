"""Per-query device counters of a config (DP load analysis): python scripts/diag_counters.py CFG METRIC"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1811_11076_b200 as t

cfg, metric = int(sys.argv[1]), sys.argv[2]
sh = t.synth_shape(cfg, 0)
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
st = t.Store(db)
idx, dist, c = t.knn(st, qs, sh["k"], metric, sh["r"])
n = sh["count"]
print("per-query counters [lb_computed, lb_pruned, full_dp, early_abandoned, gdk_calls]")
for q in range(len(qs)):
    print(q, list(map(int, c[q])))
print("sum", list(map(int, c.sum(0))), "DP'd pairs", int(c[:, 2].sum() + c[:, 3].sum()))
