"""CPU experiment: how much of the full-resolution forward / reverse LB_Box pruning does a
piecewise-aggregate (block mean) bound keep?  C5-shaped data, thresholds = true k-th distances."""
import os
import sys
import time

import numpy as np
from scipy.ndimage import maximum_filter1d, minimum_filter1d

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1811_11076_b200 as t  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8
nc = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
sh = t.synth_shape(cfg, 0)
k, r, L, d = sh["k"], sh["r"], sh["len"], sh["d"]
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
qs = qs[:nq]
orc = oracle.ref()
t0 = time.time()
oi, od, ocnt, octr = orc.knn_batch(qs, oracle.Dataset(db), k, "dtw", r, threads=os.cpu_count())
print("ref knn", time.time() - t0, "s; T =", od[:, k - 1], flush=True)
T = od[:, k - 1]
sub = db[:: max(1, db.shape[0] // nc)][:nc]


def env(x):  # x [..., L, d]
    lo = minimum_filter1d(x, 2 * r + 1, axis=-2, mode="nearest")
    hi = maximum_filter1d(x, 2 * r + 1, axis=-2, mode="nearest")
    return lo, hi


def lb(x, lo, hi):  # sum over points and dims of dist(x, [lo, hi])^2
    e = np.maximum(np.maximum(lo - x, x - hi), 0.0)
    return (e * e).sum(axis=(-1, -2))


def paa(x, w):
    s = x.shape
    return x.reshape(s[:-2] + (s[-2] // w, w, s[-1])).mean(axis=-2)


qlo, qhi = env(qs)
clo, chi = env(sub)
res = {}
for q in range(nq):
    fwd = lb(sub, qlo[q], qhi[q])
    rev = lb(qs[q], clo, chi)
    full = np.maximum(fwd, rev)
    row = {"full_pass": float((full <= T[q]).mean()), "fwd_pass": float((fwd <= T[q]).mean())}
    for w in (2, 4, 8, 16):
        f2 = w * lb(paa(sub, w), paa(qlo[q], w), paa(qhi[q], w))
        r2 = w * lb(paa(qs[q], w), paa(clo, w), paa(chi, w))
        c = np.maximum(f2, r2)
        assert (f2 <= fwd * (1 + 1e-9) + 1e-12).all() and (r2 <= rev * (1 + 1e-9) + 1e-12).all()
        row[f"paa{w}_pass"] = float((c <= T[q]).mean())
    res[q] = row
    print(q, {a: round(b, 4) for a, b in row.items()}, flush=True)
keys = res[0].keys()
print("mean", {a: round(float(np.mean([res[q][a] for q in res])), 4) for a in keys})
