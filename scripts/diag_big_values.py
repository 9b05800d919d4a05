"""Debug: the beyond-fp32-range parity cases one by one (prints progress; use with timeout)."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_1811_11076_b200 as t

rng = np.random.default_rng(41)
orc = oracle.ref() if oracle.ref_available() else oracle.port()
for scale_db, scale_q in ((1e39, 1e39), (1e39, 1.0), (1.0, 1e39), (1e200, 1e200)):
    n, L, d, r, k = 400, 40, 3, 5, 3
    X = rng.standard_normal((n, L, d)).cumsum(1)
    X[::3] *= scale_db
    Q = rng.standard_normal((4, L, d)).cumsum(1) * scale_q
    Q[1] = X[9] * (1 + 1e-9)
    Q[2] = X[10]
    ds = t.Dataset(X)
    ods = oracle.Dataset(X)
    for metric in ("dtw", "dk"):
        print("case", scale_db, scale_q, metric, "batch", flush=True)
        gi, gd, gc = t.knn(ds, Q, k, metric, r)
        for q in range(len(Q)):
            oi, od, _ = orc.knn(Q[q], ods, k, metric, r)
            keep = gi[q] != t.NO_NEIGHBOR
            ok = np.array_equal(gi[q][keep], oi) and np.array_equal(gd[q][keep], od)
            print("  q", q, "gpu", gi[q], gd[q], "ref", oi, od, "OK" if ok else "MISMATCH", gc[q], flush=True)
            print("  single", flush=True)
            rep = t.knn_dtw(Q[q], ds, k, r) if metric == "dtw" else t.knn_dk(Q[q], ds, k)
            print("  single ->", [nb.index for nb in rep.neighbors], flush=True)
