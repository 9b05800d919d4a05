"""GPU parity of the coarse LB cascade against the reference.

The DTW bound pass runs on block means of w points (w = 16 for series above 256 points with the
reverse bound on, w = 4 for shorter series on the fast path) and the DP's cumulative abandon
bounds come from block means of 4.  Every switch of the cascade must give the reference's
neighbours (indices, order, distances bit for bit) and conserved device counters
(search.hpp:10-12): cascade off, short series on the plain pass, per-point DP setup, the
guided seed sample on / off, the 1-3 query plans, lengths that are not a multiple of the
block, values beyond the fp32 range inside some blocks (NaN block means: no bound from those
blocks).  All calls go through the C ABI (libtswarp_b200.so); the checker is oracle/_ref (the
reference's own sources) or the C port.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def walks(rng, n, L, d):
    return rng.standard_normal((n, L, d)).cumsum(1)


def assert_knn_equal(gi, gd, oi, od, msg=""):
    assert np.array_equal(np.asarray(gi, dtype=np.uint64), np.asarray(oi, dtype=np.uint64)), \
        f"{msg} indices gpu={gi} oracle={oi}"
    assert np.array_equal(np.asarray(gd).view(np.uint64), np.asarray(od).view(np.uint64)), \
        f"{msg} distances gpu={gd!r} oracle={od!r}"


# (n, L, d, r, k): short series (w = 4) with and without a ragged tail, clen = 16 (the smallest
# coarse length), long series (w = 8) with a tail of 3 and the C5 shape, a band wider than the
# block and one narrower
# ... and two stores large enough for the guided seed sample (n >= 2048: the candidates with the
# smallest coarse diagonal distance instead of a strided sample), short and long series
CASES = [(400, 203, 3, 20, 3), (300, 67, 2, 9, 2), (500, 128, 3, 13, 5), (350, 256, 2, 26, 4),
         (200, 515, 2, 40, 2), (150, 1024, 3, 51, 3), (250, 96, 4, 2, 3), (300, 64, 1, 52, 1),
         (2600, 128, 3, 13, 4), (2200, 300, 2, 33, 3)]
MODES = {"default": {}, "off": {"TSW_COARSE": "0"}, "short_off": {"TSW_COARSE_SHORT": "0"},
         "pass_8_setup_8": {"TSW_COARSE_W": "8", "TSW_CSETUP_W": "8"},
         "improved_bound": {"TSW_LBI": "1"},
         "per_point_setup": {"TSW_CSETUP": "0"}, "strided_sample": {"TSW_GUIDED": "0"},
         "guided_64": {"TSW_GUIDED": "64"}}


@pytest.mark.parametrize("mode", sorted(MODES))
def test_coarse_modes_match_reference(tsw, best_oracle, mode, monkeypatch):
    import oracle

    for k_, v_ in MODES[mode].items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(1811)
    for n, L, d, r, k in CASES:
        X = walks(rng, n, L, d)
        X /= X.std(axis=1, keepdims=True)
        Q = walks(rng, 6, L, d)
        Q /= Q.std(axis=1, keepdims=True)
        Q[1] = X[7] + 1e-3 * rng.standard_normal((L, d))  # a near-duplicate: tight threshold
        Q[2] = X[11]                                       # a self-match at distance 0
        ds = tsw.Dataset(X)
        ods = oracle.Dataset(X)
        for nq in (6, 1):  # the batched plan and the reference's one-query call shape
            gi, gd, gc = tsw.knn(ds, Q[:nq], k, "dtw", r)
            for q in range(nq):
                oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
                assert_knn_equal(gi[q], gd[q], oi, od, f"{mode} n={n} L={L} d={d} r={r} nq={nq} q{q}")
                c = gc[q]
                assert c[0] == n and c[1] + c[2] + c[3] == n, (mode, n, L, c)


def test_coarse_blocks_beyond_fp32_range(tsw, best_oracle):
    """Values beyond FLT_MAX inside some blocks of some series and queries: those blocks' means
    are NaN (terms of 0) and their envelope means (0, +inf); every other block keeps its bound.
    The neighbours must be the reference's."""
    import oracle

    rng = np.random.default_rng(39)
    for n, L, d, r, k in ((300, 160, 3, 16, 3), (120, 600, 2, 40, 2)):
        X = walks(rng, n, L, d)
        X /= X.std(axis=1, keepdims=True)
        for c in range(0, n, 5):  # a few huge points in every fifth series
            X[c, rng.integers(0, L, 3), rng.integers(0, d, 3)] = 1e39 * rng.choice([-1.0, 1.0])
        Q = walks(rng, 5, L, d)
        Q /= Q.std(axis=1, keepdims=True)
        Q[1, L // 3, 0] = -3e38 * 10  # beyond the fp32 range in one block of one query
        Q[2] = X[10]
        Q[3] = X[4] + 1e-3
        ds = tsw.Dataset(X)
        ods = oracle.Dataset(X)
        gi, gd, gc = tsw.knn(ds, Q, k, "dtw", r)
        for q in range(len(Q)):
            oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
            assert_knn_equal(gi[q], gd[q], oi, od, f"n={n} L={L} q{q}")
            assert gc[q][1] + gc[q][2] + gc[q][3] == n


def test_coarse_prunes_and_reports_block(tsw, monkeypatch):
    """The cascade is what runs by default (bound_block = 4 / 16 in the plan statistics, 1 with
    TSW_COARSE=0), it prunes (lb_pruned > 0 on a clustered store), and both settings return
    the same neighbours."""
    rng = np.random.default_rng(5)
    for L, r, blk in ((128, 13, 4), (640, 40, 16)):
        X = walks(rng, 3000, L, 3)
        X /= X.std(axis=1, keepdims=True)
        Q = X[:8] + 0.05 * rng.standard_normal((8, L, 3))
        st = tsw.Store(X)
        out = {}
        for env in ("1", "0"):
            monkeypatch.setenv("TSW_COARSE", env)
            plan = tsw.Plan(st, 8, L, "dtw", r, 3)
            plan.set_queries(Q)
            plan.execute()
            idx, dist, ctr = plan.fetch()
            s = plan.stats()
            plan.close()
            assert s["bound_block"] == (blk if env == "1" else 1), s
            assert all(c[1] > 0 and c[1] + c[2] + c[3] == 3000 for c in ctr), ctr[:2]
            out[env] = (idx.copy(), dist.copy())
        assert np.array_equal(out["1"][0], out["0"][0])
        assert np.array_equal(out["1"][1].view(np.uint64), out["0"][1].view(np.uint64))
