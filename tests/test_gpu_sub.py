"""GPU parity for subsequence dog-keeper: K5 in subsequence mode against the
CPU oracle and the reference's own golden vectors.

* ``sub_dk_all`` (sparse_dk_sub for every candidate, dogkeeper.cpp:235-241): found flag,
  distance bit-exact and end column identical (earliest end on ties), for eps = +inf and
  thresholds around the distances;
* ``knn_dk_sub`` (search.cpp:250-280): neighbour indices, order and distances bit-exact;
* single-haystack ``sub_search_dk`` / ``sparse_dk_sub`` through the Python mirror.
Queries longer than one strip (64 / 128 rows) exercise the strip hand-over; haystacks shorter
than the query, ragged stores and d = 16 are covered.  All calls go through the C ABI.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def seed_sample(n):
    """Seed bounds the engine computes per query of a subsequence search (capi.cu make_plan)."""
    return min(n, 512)

HERE = os.path.dirname(os.path.abspath(__file__))
RNG = np.random.default_rng(1811_11076 + 5)
INF = float("inf")


def unhex(lst):
    return np.array([float.fromhex(v) for v in lst])


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def _check_all(tsw, port, series, q, eps):
    st = tsw.Store(series)
    found, val, end = tsw.sub_dk_all(st, q, eps)
    for i, x in enumerate(series):
        m = port.sparse_dk_sub(q, x, eps)
        if m is None:
            assert not found[i] and val[i] == INF, (i, eps, found[i], val[i])
        else:
            assert found[i], (i, eps, m)
            assert _bits(val[i]) == _bits(m[0]) and end[i] == m[1], (i, eps, val[i], end[i], m)
    return found, val


@pytest.mark.parametrize("N,L,m,d", [(200, 40, 8, 1), (200, 64, 16, 2), (150, 128, 33, 3),
                                     (100, 256, 64, 2), (60, 300, 130, 3), (40, 256, 40, 16),
                                     (20, 1024, 200, 3), (80, 20, 50, 2), (50, 70, 70, 5),
                                     (100, 1, 1, 2), (100, 5, 1, 1)])
def test_sub_dk_all_bit_exact(tsw, port, N, L, m, d):
    X = RNG.standard_normal((N, L, d)).cumsum(1)
    q = RNG.standard_normal((m, d)).cumsum(0)
    if N > 10:
        q[: min(m, L)] = X[3][: min(m, L)] + 1e-3  # a near-exact match somewhere
    _, val = _check_all(tsw, port, list(X), q, INF)
    for eps in (float(np.quantile(val, 0.1)), float(np.median(val)), 0.0):
        _check_all(tsw, port, list(X), q, eps)


def test_sub_ties_integer_grid(tsw, port):
    """Integer-valued series: many end columns share the best distance; the earliest wins."""
    X = [np.round(RNG.standard_normal((int(RNG.integers(5, 60)), 2)) * 2) for _ in range(200)]
    for m in (1, 3, 9):
        q = np.round(RNG.standard_normal((m, 2)) * 2)
        _check_all(tsw, port, X, q, INF)
        _check_all(tsw, port, X, q, 2.0)


def test_sub_ragged(tsw, port):
    X = [RNG.standard_normal((int(RNG.integers(1, 300)), 3)).cumsum(0) for _ in range(150)]
    for m in (1, 20, 100, 170):
        q = RNG.standard_normal((m, 3)).cumsum(0)
        _, val = _check_all(tsw, port, X, q, INF)
        _check_all(tsw, port, X, q, float(np.median(val)))


def test_knn_dk_sub_random(tsw, best_oracle):
    import oracle

    rng = np.random.default_rng(77)
    for trial in range(40):
        n = int(rng.integers(1, 250))
        d = int(rng.integers(1, 5))
        ragged = trial % 3 == 0
        if ragged:
            X = [rng.standard_normal((int(rng.integers(1, 120)), d)).cumsum(0) for _ in range(n)]
        else:
            L = int(rng.integers(1, 160))
            X = list(rng.standard_normal((n, L, d)).cumsum(1))
        m = int(rng.integers(1, 80))
        Q = rng.standard_normal((3, m, d)).cumsum(1)
        k = int(rng.integers(1, 12))
        ds = tsw.Dataset(X)
        gi, gd, gc = tsw.knn(ds, Q, k, "dk_sub")
        ods = oracle.Dataset(X)
        for q in range(len(Q)):
            oi, od, _ = best_oracle.knn(Q[q], ods, k, "dk_sub")
            assert np.array_equal(gi[q], oi), (trial, q, gi[q], oi)
            assert np.array_equal(_bits(gd[q]), _bits(od)), (trial, q, gd[q], od)
            assert gc[q][4] == seed_sample(n) and gc[q][2] + gc[q][3] == n


def test_knn_dk_sub_box_bound_cases(tsw, best_oracle, monkeypatch):
    """The subsequence box bound (per-tile bounding boxes of the store against eight query
    points, fp32 interval arithmetic) only prunes: with it on and off the neighbours equal the
    reference's, on ragged stores, d = 1..5 (d >= 5: the fp64 form), query subsequences cut out
    of stored series (distance 0 and near 0: the tightest thresholds), series shorter than the
    query, and values beyond the fp32 range."""
    import oracle

    rng = np.random.default_rng(1234)
    for trial in range(12):
        d = 1 + trial % 5
        n = int(rng.integers(60, 400))
        X = [rng.standard_normal((int(rng.integers(3, 300)), d)).cumsum(0) for _ in range(n)]
        if trial % 4 == 3:
            for c in range(0, n, 7):
                X[c] = X[c] * 1e39  # beyond the fp32 range: boxes with infinite sides
        m = int(rng.integers(8, 90))
        Q = rng.standard_normal((4, m, d)).cumsum(1)
        src = [x for x in X if len(x) >= m + 5]
        if src:
            Q[0] = src[0][3:3 + m]                                       # an exact subsequence
            Q[1] = src[-1][2:2 + m] + 1e-4 * rng.standard_normal((m, d))  # a near one
        k = int(rng.integers(1, 8))
        ods = oracle.Dataset(X)
        want = [best_oracle.knn(Q[q], ods, k, "dk_sub") for q in range(len(Q))]
        for box in ("1", "0"):
            monkeypatch.setenv("TSW_SUB_BOX", box)
            gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dk_sub")
            for q in range(len(Q)):
                oi, od, _ = want[q]
                assert np.array_equal(gi[q], oi), (trial, box, q, gi[q], oi)
                assert np.array_equal(_bits(gd[q]), _bits(od)), (trial, box, q, gd[q], od)
                assert gc[q][2] + gc[q][3] == n


def test_knn_dk_sub_large_k_and_dupes(tsw, best_oracle):
    import oracle

    base = list(RNG.standard_normal((30, 90, 2)).cumsum(1))
    X = base + base  # duplicate haystacks: equal distances, lower index first
    q = base[4][10:40] + 0.01
    for k in (1, 5, 33, 64, 65, 100):
        gi, gd, _ = tsw.knn(tsw.Dataset(X), q[None], k, "dk_sub")
        oi, od, _ = best_oracle.knn(q, oracle.Dataset(X), k, "dk_sub")
        assert np.array_equal(gi[0], oi) and np.array_equal(_bits(gd[0]), _bits(od)), k


def test_sub_golden_reference_vectors(tsw):
    """The reference's own outputs (tests/golden/reference_sub_vectors.json)."""
    with open(os.path.join(HERE, "golden", "reference_sub_vectors.json")) as f:
        golden = json.load(f)
    for case in golden["cases"]:
        d = case["d"]
        series = [unhex(s).reshape(-1, d) for s in case["series"]]
        queries = [unhex(q).reshape(-1, d) for q in case["queries"]]
        ds = tsw.Dataset(series)
        for e in case["knn"]:
            rep = tsw.knn_dk_sub(queries[e["q"]], ds, e["k"])
            assert [nb.index for nb in rep.neighbors] == e["index"], (case["name"], e)
            assert [nb.distance.hex() for nb in rep.neighbors] == e["distance"], (case["name"], e)
            assert rep.counters.gdk_calls == seed_sample(len(series))  # seed bounds computed
        st = tsw.Store(series[:10])
        for qi, q in enumerate(queries):
            found, val, end = tsw.sub_dk_all(st, q, INF)
            for e in (e for e in case["pair"] if e["q"] == qi):
                assert found[e["i"]] and [val[e["i"]].hex(), int(end[e["i"]])] == e["sub_inf"]
                m = tsw.sparse_dk_sub(q, series[e["i"]], float.fromhex(e["sub_inf"][0]) * 0.999)
                assert (None if m is None else [m.distance.hex(), m.end_index]) == e["sub_below"]
                m = tsw.sub_search_dk(q, series[e["i"]], float.fromhex(e["sub_inf"][0]))
                assert (None if m is None else [m.distance.hex(), m.end_index]) == e["search_at"]


def test_sub_errors_mirror_reference(tsw):
    X = RNG.standard_normal((5, 12, 2))
    ds = tsw.Dataset(X)
    with pytest.raises(ValueError, match="knn_dk_sub: k must be positive"):
        tsw.knn_dk_sub(X[0], ds, 0)
    with pytest.raises(ValueError, match="dimensionality mismatch"):
        tsw.sub_search_dk(np.zeros((3, 3)), X[0])
    with pytest.raises(ValueError, match="eps must be nonnegative"):
        tsw.sparse_dk_sub(X[0][:3], X[1], -1.0)


def test_knn_dk_sub_deep_queue_claims(tsw, best_oracle):
    """A queue deep enough (64 queries x 6000 series = 384k pairs) that the DP warps claim 8
    slots per atomic and compute the row-0 liveness bits of a claim's pairs in one pass over
    the shared series (claims that straddle two series take the per-pair path): the neighbours
    of a sample of queries equal the reference's, bit for bit."""
    import oracle

    rng = np.random.default_rng(4242)
    n, L, m, d, k = 6000, 64, 16, 2, 3
    X = list(rng.standard_normal((n, L, d)).cumsum(1))
    Q = rng.standard_normal((64, m, d)).cumsum(1)
    Q[5] = X[123][10:10 + m] + 1e-3 * rng.standard_normal((m, d))
    gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dk_sub")
    ods = oracle.Dataset(X)
    for q in (0, 5, 17, 31, 40, 63):
        oi, od, _ = best_oracle.knn(Q[q], ods, k, "dk_sub")
        assert np.array_equal(gi[q], oi), (q, gi[q], oi)
        assert np.array_equal(_bits(gd[q]), _bits(od)), (q, gd[q], od)
        assert gc[q][4] == seed_sample(n) and gc[q][2] + gc[q][3] == n
