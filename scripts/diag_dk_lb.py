"""CPU experiment: pruning of cheap DK (discrete Frechet) lower bounds at the true k-th distance."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1811_11076_b200 as t  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sh = t.synth_shape(cfg, 0)
k = sh["k"]
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
qs = qs[:nq]
orc = oracle.ref()
t0 = time.time()
oi, od, ocnt, octr = orc.knn_batch(qs, oracle.Dataset(db), k, "dk", 0, threads=os.cpu_count())
T = od[:, k - 1]
print("ref knn_dk", round(time.time() - t0, 1), "s; T =", np.round(T, 3), flush=True)
cmax, cmin = db.max(axis=1), db.min(axis=1)  # [n, d]
amax, amin = db.argmax(axis=1), db.argmin(axis=1)
for q in range(nq):
    x = qs[q]
    ends = np.maximum(np.linalg.norm(db[:, 0] - x[0], axis=1), np.linalg.norm(db[:, -1] - x[-1], axis=1))
    ext = np.maximum(np.abs(cmax - x.max(axis=0)), np.abs(cmin - x.min(axis=0))).max(axis=1)
    p0 = (ends <= T[q]).mean()
    p1 = ((ends <= T[q]) & (ext <= T[q])).mean()
    print(q, "ends pass", round(float(p0), 4), "ends+extent pass", round(float(p1), 4), flush=True)
