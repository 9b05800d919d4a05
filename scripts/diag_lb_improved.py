"""CPU experiment: how many of the pairs that pass max(forward, reverse) LB_Box would a
two-pass LB_Improved-style bound (Lemire 2009, per dimension on the box envelopes) remove, at
the true k-th distances?  C5-shaped data."""
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
k, r = sh["k"], sh["r"]
db, _ = t.synth(cfg, 0)
qs, _ = t.synth(cfg, 1)
qs = qs[:nq]
orc = oracle.ref()
oi, od, ocnt, octr = orc.knn_batch(qs, oracle.Dataset(db), k, "dtw", r, threads=os.cpu_count())
T = od[:, k - 1]
sub = db[:: max(1, db.shape[0] // nc)][:nc]


def env(x):
    return (minimum_filter1d(x, 2 * r + 1, axis=-2, mode="nearest"),
            maximum_filter1d(x, 2 * r + 1, axis=-2, mode="nearest"))


def lb(x, lo, hi):
    e = np.maximum(np.maximum(lo - x, x - hi), 0.0)
    return (e * e).sum(axis=(-1, -2))


qlo, qhi = env(qs)
clo, chi = env(sub)
tot = {"two_sided": 0.0, "improved_fwd": 0.0, "improved_both": 0.0}
for q in range(nq):
    fwd = lb(sub, qlo[q], qhi[q])
    rev = lb(qs[q], clo, chi)
    two = np.maximum(fwd, rev)
    keep = two <= T[q]
    idx = np.nonzero(keep)[0]
    # LB_Improved(c, q) = LB(c; env q) + LB(q; env(H)), H = projection of c on env q
    H = np.clip(sub[idx], qlo[q], qhi[q])
    hlo, hhi = env(H)
    imp_f = fwd[idx] + lb(qs[q], hlo, hhi)
    # ... and with the roles swapped: project q on env c, then c against env of that
    G = np.clip(qs[q][None], clo[idx], chi[idx])
    glo, ghi = env(G)
    imp_r = rev[idx] + lb(sub[idx], glo, ghi)
    p_two = keep.mean()
    p_f = (imp_f <= T[q]).sum() / len(sub)
    p_b = (np.maximum(imp_f, imp_r) <= T[q]).sum() / len(sub)
    print(q, "two-sided pass", round(float(p_two), 4), "improved (fwd)", round(float(p_f), 4),
          "improved (both)", round(float(p_b), 4), flush=True)
    tot["two_sided"] += p_two / nq
    tot["improved_fwd"] += p_f / nq
    tot["improved_both"] += p_b / nq
print("mean", {a: round(float(b), 4) for a, b in tot.items()})


# ---- a block-level relaxation: everything from per-block means / minima / maxima ----------------
def blk(x, w, f):
    s_ = x.shape
    return f(x.reshape(s_[:-2] + (s_[-2] // w, w, s_[-1])), axis=-2)


def coarse_improved(w):
    L = sub.shape[1]
    nb = L // w
    cmean, cmn, cmx = blk(sub, w, np.mean), blk(sub, w, np.min), blk(sub, w, np.max)
    res = 0.0
    rb = (r + w - 1) // w  # blocks a window of radius r can reach on either side
    for q in range(nq):
        lq_mean, uq_mean = blk(qlo[q], w, np.mean), blk(qhi[q], w, np.mean)
        lq_mn, lq_mx = blk(qlo[q], w, np.min), blk(qlo[q], w, np.max)
        uq_mn, uq_mx = blk(qhi[q], w, np.min), blk(qhi[q], w, np.max)
        qmean = blk(qs[q], w, np.mean)
        f1 = w * lb(cmean, lq_mean, uq_mean)                      # Jensen on the first term
        hlo = np.maximum(lq_mn, np.minimum(cmn, uq_mn))           # H_j >= hlo_B on block B
        hhi = np.minimum(uq_mx, np.maximum(cmx, lq_mx))           # H_j <= hhi_B
        elo = minimum_filter1d(hlo, 2 * rb + 1, axis=-2, mode="nearest")
        ehi = maximum_filter1d(hhi, 2 * rb + 1, axis=-2, mode="nearest")
        f2 = w * lb(qmean, elo, ehi)                              # Jensen in q, block-constant interval
        rev = w * lb(qmean, blk(clo, w, np.mean), blk(chi, w, np.mean))
        key = np.maximum(f1 + f2, rev)
        res += (key <= T[q]).mean() / nq
    return res


for w in (4, 8):
    print("block-level improved, w =", w, "pass", round(float(coarse_improved(w)), 4))
