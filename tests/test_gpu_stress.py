"""Randomised GPU-vs-oracle stress over the pruning logic that is hardest to get right: DK
strips restarting at live boundary cells (queries spanning several 64/128-row strips, ragged
stores, class-structured data with narrow corridors), subsequence DK, and DTW with the
cumulative bound.  Every answer -- indices, order, distance bits -- must equal the C port of
the reference (oracle/tswarp_oracle.c), which tests/test_oracle.py pins to the reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _corridor_data(rng, n, L, d):
    """warped copies of a few smooth prototypes: near neighbours with narrow DP corridors"""
    protos = rng.standard_normal((4, L, d)).cumsum(1)
    out = np.empty((n, L, d))
    t = np.arange(L)
    for i in range(n):
        p = protos[i % 4]
        warp = np.clip(t + rng.integers(-3, 4) + 3 * np.sin(t / (5 + i % 7)), 0, L - 1)
        for k in range(d):
            out[i, :, k] = np.interp(warp, t, p[:, k])
    return out + 0.05 * rng.standard_normal((n, L, d))


@pytest.mark.parametrize("seed", range(6))
def test_stress_dk_multi_strip(tsw, port, seed):
    import oracle

    rng = np.random.default_rng(1000 + seed)
    for trial in range(6):
        d = int(rng.integers(1, 4))
        if trial % 2:
            X = _corridor_data(rng, int(rng.integers(20, 120)), int(rng.integers(70, 260)), d)
            series = list(X)
        else:
            series = [rng.standard_normal((int(rng.integers(1, 260)), d)).cumsum(0)
                      for _ in range(int(rng.integers(20, 120)))]
        m = int(rng.integers(65, 300))
        src = series[int(rng.integers(0, len(series)))]
        near = np.resize(src[: min(len(src), 40)].repeat(4, 0), (m, d))  # slowed-down stored shape
        Q = np.stack([near + 0.05 * rng.standard_normal((m, d)), rng.standard_normal((m, d)).cumsum(0)])
        ds, ods = tsw.Dataset(series), oracle.Dataset(series)
        k = int(rng.integers(1, 9))
        for metric in ("dk", "dk_sub"):
            gi, gd, gc = tsw.knn(ds, Q, k, metric)
            for q in range(len(Q)):
                oi, od, _ = port.knn(Q[q], ods, k, metric)
                assert np.array_equal(gi[q], oi), (seed, trial, metric, q, gi[q], oi)
                assert np.array_equal(gd[q].view(np.uint64), od.view(np.uint64)), (seed, trial, metric, q)
                assert gc[q][2] + gc[q][3] == len(series)


@pytest.mark.parametrize("seed", range(4))
def test_stress_dtw(tsw, port, seed):
    import oracle

    rng = np.random.default_rng(2000 + seed)
    for trial in range(6):
        d = int(rng.integers(1, 7))
        L = int(rng.integers(2, 200))
        r = int(rng.integers(0, min(L, 40)))
        X = _corridor_data(rng, int(rng.integers(10, 150)), L, d)
        Q = np.stack([X[1] + 0.01 * rng.standard_normal((L, d)), rng.standard_normal((L, d)).cumsum(0)])
        k = int(rng.integers(1, 9))
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
        for q in range(len(Q)):
            oi, od, _ = port.knn(Q[q], oracle.Dataset(X), k, "dtw", r)
            assert np.array_equal(gi[q], oi), (seed, trial, q, L, d, r, gi[q], oi)
            assert np.array_equal(gd[q].view(np.uint64), od.view(np.uint64)), (seed, trial, q)
            assert gc[q][1] + gc[q][2] + gc[q][3] == len(X)
