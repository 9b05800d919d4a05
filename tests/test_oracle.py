"""CPU: pin the oracle before trusting it.

* the C port (oracle/tswarp_oracle.c) against the SPEC.md known-answer examples (kat.json),
* the C port against golden vectors produced by the reference itself
  (tests/golden/reference_vectors.json, made by tests/golden/make_golden.py from oracle/_ref),
* the C port against the live reference library (oracle/_ref) on seeded random inputs when it
  is built, and the SPEC acceptance properties 2, 3, 4, 5 and 8.
"""
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
INF = float("inf")


def num(v):
    return INF if v == "inf" else float(v)


def arr(x):
    return np.asarray(x, dtype=np.float64)


def unhex(lst):
    return np.array([float.fromhex(v) for v in lst])


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(HERE, "golden", "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "reference_vectors.json")) as f:
        return json.load(f)


def oracles():
    out = [oracle.port()]
    if oracle.ref_available() or os.path.isdir(oracle.REF_ROOT):
        try:
            out.append(oracle.ref())
        except Exception:
            pass
    return out


# ---- SPEC known answers --------------------------------------------------------------
@pytest.mark.parametrize("which", [0, 1])
def test_spec_kats(kat, which):
    os_ = oracles()
    if which >= len(os_):
        pytest.skip("reference library not available")
    O = os_[which]
    for e in kat["envelope"]:
        lo, hi = O.envelope(arr(e["t"]), e["r"])
        assert lo.tolist() == e["lower"] and hi.tolist() == e["upper"], e["spec"]
    for e in kat["lb_box"]:
        assert O.lb_box(arr(e["candidate"]), arr(e["query"]), e["r"]) == e["value"], e["spec"]
    for e in kat["lb_sigma_min"]:
        assert O.lb_sigma_min(arr(e["s"]), arr(e["t"]), e["r"]) == e["value"], e["spec"]
    for e in kat["dtw_banded"]:
        assert O.dtw_banded(arr(e["s"]), arr(e["t"]), e["r"]) == num(e["value"]), e["spec"]
    for e in kat["dtw_early_abandon"]:
        assert O.dtw_early_abandon(arr(e["s"]), arr(e["t"]), e["r"], num(e["eps"])) == \
            (e["exact"], num(e["value"])), e["spec"]
    for e in kat["dk_full"]:
        assert O.dk_full(arr(e["s"]), arr(e["t"])) == e["value"], e["spec"]
    for e in kat["gdk"]:
        assert O.gdk(arr(e["s"]), arr(e["t"]), num(e["eps"])) == e["value"], e["spec"]
    for e in kat["sparse_dk"]:
        assert O.sparse_dk(arr(e["s"]), arr(e["t"]), num(e["eps"])) == \
            (e["exact"], num(e["value"])), e["spec"]
    for e in kat["znormalize"]:
        assert O.znormalize(arr(e["s"])).tolist() == e["value"], e["spec"]
    for e in kat["knn"]:
        idx, dist, _ = O.knn(arr(e["query"]), oracle.Dataset(arr(e["data"])), e["k"], e["metric"], e["r"])
        assert idx.tolist() == e["index"] and dist.tolist() == e["distance"], e["spec"]


# ---- golden vectors produced by the reference ---------------------------------------------
def _case_data(case):
    d = case["d"]
    series = [unhex(s).reshape(-1, d) for s in case["series"]]
    queries = [unhex(q).reshape(-1, d) for q in case["queries"]]
    return series, queries


def test_port_matches_reference_golden(golden):
    P = oracle.port()
    for case in golden["cases"]:
        series, queries = _case_data(case)
        ds = oracle.Dataset(series)
        r = case["r"]
        for e in case["knn"]:
            idx, dist, ctr = P.knn(queries[e["q"]], ds, e["k"], e["metric"], r)
            assert idx.tolist() == e["index"], (case["name"], e)
            assert [v.hex() for v in dist.tolist()] == e["distance"], (case["name"], e)
            assert ctr.tolist() == e["counters"], (case["name"], e)
        for e in case["epsnn"]:
            idx, dist, _ = P.epsnn_dk(queries[e["q"]], ds, float.fromhex(e["eps"]))
            assert idx.tolist() == e["index"] and [v.hex() for v in dist.tolist()] == e["distance"]
        q = queries[0]
        for e in case["pair"]:
            s = series[e["i"]]
            assert P.dk_full(q, s).hex() == e["dk_full"]
            assert P.gdk(q, s).hex() == e["gdk"]
            ex, v = P.sparse_dk(q, s, P.dk_full(q, s) * 0.999)
            assert [ex, v.hex()] == e["sparse_dk_below"]
            if not case["ragged"]:
                assert P.dtw_banded(q, s, r).hex() == e["dtw_banded"]
                ex, v = P.dtw_early_abandon(q, s, r, P.dtw_banded(q, s, r))
                assert [ex, v.hex()] == e["dtw_early_abandon_at_d"]
                assert P.lb_box(s, q, r).hex() == e["lb_box"]
        if not case["ragged"]:
            lo, hi = P.envelope(q, r)
            assert [v.hex() for v in lo.ravel()] == case["envelope_q0"]["lo"]
            assert [v.hex() for v in hi.ravel()] == case["envelope_q0"]["hi"]
            assert [v.hex() for v in P.znormalize(q).ravel()] == case["znormalize_q0"]


def test_port_matches_live_reference():
    if not (oracle.ref_available() or os.path.isdir(oracle.REF_ROOT)):
        pytest.skip("reference library not available")
    P, R = oracle.port(), oracle.ref()
    rng = np.random.default_rng(5)
    for _ in range(300):
        d = int(rng.integers(1, 5))
        m = int(rng.integers(1, 24))
        n = int(rng.integers(1, 24))
        r = int(rng.integers(0, 26))
        s = rng.standard_normal((m, d)).cumsum(0)
        t = rng.standard_normal((n, d)).cumsum(0)
        eps = float(rng.random() * 4)
        assert P.dtw_banded(s, t, r) == R.dtw_banded(s, t, r)
        assert P.dk_full(s, t) == R.dk_full(s, t)
        assert P.gdk(s, t, eps) == R.gdk(s, t, eps)
        assert P.sparse_dk(s, t, eps) == R.sparse_dk(s, t, eps)
        if m == n:
            assert P.lb_box(t, s, r) == R.lb_box(t, s, r)
            assert P.dtw_early_abandon(s, t, r, eps * 10) == R.dtw_early_abandon(s, t, r, eps * 10)
    for _ in range(30):
        d = int(rng.integers(1, 4))
        L = int(rng.integers(1, 30))
        n = int(rng.integers(1, 120))
        r = int(rng.integers(0, 8))
        k = int(rng.integers(1, 10))
        X = rng.standard_normal((n, L, d)).cumsum(1)
        q = rng.standard_normal((L, d)).cumsum(0)
        ds = oracle.Dataset(X)
        for metric in ("dtw", "dk"):
            a, b = P.knn(q, ds, k, metric, r), R.knn(q, ds, k, metric, r)
            assert all(np.array_equal(x, y) for x, y in zip(a, b))


# ---- SPEC acceptance properties on the port ------------------------------
def test_acceptance_2_3_4_dk():
    P = oracle.port()
    rng = np.random.default_rng(2)
    for _ in range(400):
        d = int(rng.integers(1, 8))
        s = rng.standard_normal((int(rng.integers(1, 40)), d))
        t = rng.standard_normal((int(rng.integers(1, 40)), d))
        full = P.dk_full(s, t)
        assert P.sparse_dk(s, t, INF) == (True, full)                # criterion 2
        eps = float(rng.random() * 3)
        ex, v = P.sparse_dk(s, t, eps)                                 # criterion 3
        assert (ex and v == full and full <= eps) or (not ex and full > eps)
        assert P.gdk(s, t) >= full                                     # criterion 4


def test_acceptance_5_lower_bound_chain():
    P = oracle.port()
    rng = np.random.default_rng(3)
    for _ in range(400):
        d = int(rng.choice([1, 2, 4, 8]))
        n = int(rng.integers(1, 30))
        r = int(rng.integers(0, 8))
        s = rng.standard_normal((n, d))
        t = rng.standard_normal((n, d))
        lb = P.lb_box(s, t, r)       # lb_box(s, envelope(t, r))
        sig = P.lb_sigma_min(s, t, r)
        dtw = P.dtw_banded(s, t, r)
        assert lb <= sig * (1 + 1e-9) and sig <= dtw * (1 + 1e-9)


def test_acceptance_8_search_equals_brute_force():
    P = oracle.port()
    rng = np.random.default_rng(4)
    for _ in range(40):
        n = int(rng.integers(1, 80))
        L = int(rng.integers(1, 32))
        d = int(rng.integers(1, 4))
        r = int(rng.integers(0, 6))
        k = int(rng.integers(1, 8))
        X = rng.standard_normal((n, L, d)).cumsum(1)
        q = rng.standard_normal((L, d)).cumsum(0)
        ds = oracle.Dataset(X)
        for metric, allv in (("dtw", P.dtw_all(q, ds, r)), ("dk", P.dk_all(q, ds))):
            order = sorted(range(n), key=lambda i: (allv[i], i))[:min(k, n)]
            idx, dist, _ = P.knn(q, ds, k, metric, r)
            assert idx.tolist() == order and dist.tolist() == [allv[i] for i in order]


# ---- subsequence DK ----------------------------------------------------
@pytest.fixture(scope="module")
def golden_sub():
    with open(os.path.join(HERE, "golden", "reference_sub_vectors.json")) as f:
        return json.load(f)


def sub_case_data(case):
    d = case["d"]
    series = [unhex(s).reshape(-1, d) for s in case["series"]]
    queries = [unhex(q).reshape(-1, d) for q in case["queries"]]
    return series, queries


def _hx_match(m):
    return None if m is None else [m[0].hex(), m[1]]


def test_port_matches_reference_sub_golden(golden_sub):
    P = oracle.port()
    for case in golden_sub["cases"]:
        series, queries = sub_case_data(case)
        ds = oracle.Dataset(series)
        for e in case["knn"]:
            idx, dist, ctr = P.knn(queries[e["q"]], ds, e["k"], "dk_sub")
            assert idx.tolist() == e["index"], (case["name"], e)
            assert [v.hex() for v in dist.tolist()] == e["distance"], (case["name"], e)
            assert ctr.tolist() == e["counters"], (case["name"], e)
        for e in case["pair"]:
            q, x = queries[e["q"]], series[e["i"]]
            full = P.sparse_dk_sub(q, x, INF)
            assert _hx_match(full) == e["sub_inf"]
            assert _hx_match(P.gdk_sub(q, x)) == e["gdk_sub"]
            assert _hx_match(P.sparse_dk_sub(q, x, full[0] * 0.999)) == e["sub_below"]
            assert _hx_match(P.sub_search_dk(q, x, full[0])) == e["search_at"]
            assert P.dk_sub_full(q, x) == full  # brute force: same value and end column


def test_port_sub_matches_live_reference():
    if not (oracle.ref_available() or os.path.isdir(oracle.REF_ROOT)):
        pytest.skip("reference library not available")
    P, R = oracle.port(), oracle.ref()
    rng = np.random.default_rng(12)
    for it in range(600):
        d = int(rng.integers(1, 5))
        m, n = int(rng.integers(1, 20)), int(rng.integers(1, 40))
        s = rng.standard_normal((m, d)).cumsum(0)
        t = rng.standard_normal((n, d)).cumsum(0)
        if it % 7 == 0:  # integer grids: many exact ties between end columns
            s, t = np.round(s), np.round(t)
        eps = float(rng.random() * 4)
        assert P.sparse_dk_sub(s, t, eps) == R.sparse_dk_sub(s, t, eps)
        assert P.sub_search_dk(s, t, eps) == R.sub_search_dk(s, t, eps)
        assert P.gdk_sub(s, t, eps) == R.gdk_sub(s, t, eps)
    for _ in range(20):
        d = int(rng.integers(1, 4))
        n = int(rng.integers(1, 80))
        X = [rng.standard_normal((int(rng.integers(1, 50)), d)).cumsum(0) for _ in range(n)]
        q = rng.standard_normal((int(rng.integers(1, 15)), d)).cumsum(0)
        k = int(rng.integers(1, 8))
        ds = oracle.Dataset(X)
        a, b = P.knn(q, ds, k, "dk_sub"), R.knn(q, ds, k, "dk_sub")
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_sub_properties():
    """sub <= whole DK (the whole path is one subsequence path), the sparse engine equals the
    brute-force DP, and knn_dk_sub equals the brute-force (distance, index) top-k."""
    P = oracle.port()
    rng = np.random.default_rng(13)
    for _ in range(300):
        d = int(rng.integers(1, 4))
        s = rng.standard_normal((int(rng.integers(1, 25)), d))
        t = rng.standard_normal((int(rng.integers(1, 40)), d))
        full = P.dk_sub_full(s, t)
        assert P.sparse_dk_sub(s, t, INF) == full
        assert full[0] <= P.dk_full(s, t)
        g, _ = P.gdk_sub(s, t)
        assert g >= full[0]
    X = [rng.standard_normal((int(rng.integers(5, 60)), 2)).cumsum(0) for _ in range(120)]
    ds = oracle.Dataset(X)
    for _ in range(5):
        q = rng.standard_normal((int(rng.integers(2, 12)), 2)).cumsum(0)
        allv = [P.dk_sub_full(q, x)[0] for x in X]
        order = sorted(range(len(X)), key=lambda i: (allv[i], i))[:4]
        idx, dist, ctr = P.knn(q, ds, 4, "dk_sub")
        assert idx.tolist() == order and dist.tolist() == [allv[i] for i in order]
        assert ctr[4] == len(X) and ctr[2] + ctr[3] == len(X)
