"""Diagnostic: plan (device queries) vs tsw_knn (host queries) vs GPU brute force for one config."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_11076_b200 as t  # noqa: E402

cfg, metric = int(sys.argv[1]), sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sh = t.synth_shape(cfg, 0)
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
st = t.Store(db)
k, r = sh["k"], sh["r"]
res = []
for i in range(reps):
    res.append(t.knn(st, qs, k, metric, r))
bad = set()
for i in range(1, reps):
    for q in range(len(qs)):
        if not (np.array_equal(res[i][0][q], res[0][0][q]) and np.array_equal(res[i][1][q], res[0][1][q])):
            bad.add(q)
print("mismatching queries:", sorted(bad))
for q in sorted(bad)[:4]:
    ex, val = t.dist_all(st, qs[q], metric, r)
    order = sorted(range(len(db)), key=lambda i: (val[i], i))[:k]
    print("q", q, "brute", order, [val[i] for i in order])
    for i in range(reps):
        print("   run", i, res[i][0][q].tolist(), res[i][1][q].tolist())
