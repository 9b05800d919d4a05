"""GPU parity: every kernel and both k-NN drivers against the CPU oracle on the same inputs.

Bar (BASELINE.json north_star): neighbour indices and order bit-exact under the (distance,
index) tie rule; DK distances bit-exact; DTW distances bit-exact (allowed: 1e-12 relative,
asserted exactly here because the suffix-order recursion is reproduced).
The pipeline's LB_Box is an fp32 directed-rounding LOWER bound of the reference's value (checked
lb <= oracle, and within rel. 2e-5 of it); the fp64 restatement tsw_lb_box_exact_all is compared
with the reference bit for bit.  All calls go through the C ABI (libtswarp_b200.so).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def seed_sample(n, L=None, d=1, k=1, nq=4):
    """Seed bounds the engine computes per query (capi.cu make_plan).  Strided sample: 2048,
    ~n/24 for n >= 96k.  Guided sample (whole-match DK on a uniform store of the query's length
    L, n >= 2048, k <= 32, >= 4 queries or n >= 98304, the estimate's shared-memory tile fits):
    the 32 best-ranked candidates."""
    if L is not None and n >= 2048 and k <= 32 and (nq >= 4 or n >= 98304):
        w2 = 1
        while w2 * 2 * 24 <= L:
            w2 *= 2
        clen2 = L // w2
        if clen2 >= 8 and (clen2 + 31) // 32 * 32 * d * 101 * 4 <= 96 * 1024:
            return 32
    return min(n, 2048 if n < 98304 else min(8192, n // 24))

RNG = np.random.default_rng(20181127)


def walks(rng, n, L, d):
    return rng.standard_normal((n, L, d)).cumsum(1)


def assert_knn_equal(gi, gd, oi, od, msg=""):
    assert np.array_equal(np.asarray(gi, dtype=np.uint64), np.asarray(oi, dtype=np.uint64)), \
        f"{msg} indices gpu={gi} oracle={oi}"
    assert np.array_equal(np.asarray(gd).view(np.uint64), np.asarray(od).view(np.uint64)), \
        f"{msg} distances gpu={gd!r} oracle={od!r}"


# ---- K1 envelope ------------------------------------------------------------------------
@pytest.mark.parametrize("L,d,r", [(1, 1, 0), (3, 1, 1), (17, 3, 0), (64, 2, 5), (128, 3, 13),
                                   (50, 4, 100), (256, 16, 26)])
def test_envelope_exact(tsw, port, L, d, r):
    s = RNG.standard_normal((L, d)).cumsum(0)
    lo, hi = tsw.envelope(s, r)
    olo, ohi = port.envelope(s, r)
    assert np.array_equal(lo, olo) and np.array_equal(hi, ohi)


def test_envelope_spec_kat(tsw):
    # t=((1),(3),(2)), r=1 -> lower ((1),(1),(2)), upper ((3),(3),(3))
    lo, hi = tsw.envelope(np.array([[1.0], [3.0], [2.0]]), 1)
    assert lo.ravel().tolist() == [1, 1, 2] and hi.ravel().tolist() == [3, 3, 3]


# ---- K2 LB_Box + seed upper bound --------------------------------------------------------
@pytest.mark.parametrize("N,L,d,r", [(300, 32, 1, 3), (500, 64, 3, 6), (200, 128, 2, 13),
                                     (100, 256, 16, 26), (64, 33, 3, 4), (50, 1, 2, 0)])
def test_lb_box_all(tsw, port, N, L, d, r):
    X = walks(RNG, N, L, d)
    q = walks(RNG, 1, L, d)[0]
    lb, ub = tsw.lb_box_all(tsw.Store(X), q, r)
    olb = np.array([port.lb_box(X[i], q, r) for i in range(N)])
    # K2 runs in fp32 with directed rounding: a rigorous lower bound of the fp64 LB_Box that is
    # tight to fp32 precision
    assert np.all(lb <= olb), "fp32 LB_Box above the reference lb_box"
    np.testing.assert_allclose(lb, olb, rtol=2e-5, atol=1e-6)
    dtw = np.array([port.dtw_banded(q, X[i], r) for i in range(N)])
    assert np.all(ub >= dtw), "diagonal upper bound below computed DTW"
    assert np.all(lb <= dtw * (1 + 1e-12)), "LB_Box above DTW"


def test_lb_box_sneak_past(tsw, port):
    # SPEC.md:144-147 Fig. 3: t=((0,1),(0,0),(1,0)), r=2, s=((1,1),(1,1),(1,1)) -> lb_box 0 < dtw
    t = np.array([[0.0, 1.0], [0.0, 0.0], [1.0, 0.0]])
    s = np.ones((3, 2))
    lb, _ = tsw.lb_box_all(tsw.Store(s[None]), t, 2)
    assert lb[0] == 0.0
    ex, val = tsw.dist_all(tsw.Store(s[None]), t, "dtw", 2)
    assert ex[0] and val[0] == port.dtw_banded(t, s, 2) and val[0] > 0


# ---- K4 DTW DP ---------------------------------------------------------------------------
@pytest.mark.parametrize("N,L,d,r", [(200, 1, 1, 0), (200, 2, 1, 1), (300, 16, 2, 0),
                                     (300, 40, 3, 3), (300, 64, 1, 64), (200, 128, 3, 13),
                                     (100, 256, 2, 26), (60, 256, 16, 26), (40, 97, 5, 40),
                                     (20, 300, 3, 70), (10, 1024, 3, 51), (16, 200, 2, 150)])
def test_dtw_all_bit_exact(tsw, port, N, L, d, r):
    X = walks(RNG, N, L, d)
    q = walks(RNG, 1, L, d)[0]
    st = tsw.Store(X)
    ex, val = tsw.dist_all(st, q, "dtw", r)
    ref = port.dtw_all(q, __import__("oracle").Dataset(X), r)
    assert ex.all()
    assert np.array_equal(val.view(np.uint64), ref.view(np.uint64))
    # thresholded: Exact iff d <= eps (dtw_early_abandon, dtw.cpp:82-90)
    eps = float(np.median(ref))
    ex2, val2 = tsw.dist_all(st, q, "dtw", r, eps)
    for i in range(N):
        oe, ov = port.dtw_early_abandon(q, X[i], r, eps)
        assert ex2[i] == oe and val2[i] == ov, (i, ex2[i], val2[i], oe, ov)


@pytest.mark.parametrize("variant", ["1,16", "1,32", "2,8", "2,16", "2,32", "generic"])
def test_dtw_fast_path_variants(tsw, port, variant, monkeypatch):
    """Every (cells per lane G, group width WL) instance of the guarded fast path
    (kernels_dtw4.cu) and the generic kernel, d = 1..4, bands that put offset +r on either
    lane parity and every band radius mod 4, L not a multiple of the 32-point tile (padding =
    guard values)."""
    import oracle

    if variant == "generic":
        monkeypatch.setenv("TSW_DTW_GENERIC", "1")
    else:
        monkeypatch.setenv("TSW_DTW4", variant)
    rng = np.random.default_rng(12)
    for d in (1, 2, 3, 4):
        for L, r in ((1, 0), (5, 2), (37, 6), (45, 7), (60, 9), (70, 14), (70, 15), (90, 13),
                     (80, 25), (100, 27), (100, 30), (120, 52)):
            X = walks(rng, 24, L, d)
            q = walks(rng, 1, L, d)[0]
            ex, val = tsw.dist_all(tsw.Store(X), q, "dtw", r)
            ref = port.dtw_all(q, oracle.Dataset(X), r)
            assert ex.all() and np.array_equal(val.view(np.uint64), ref.view(np.uint64)), (d, L, r)
            Q = np.concatenate([q[None], X[3:4] + 1e-3])
            gi, gd, _ = tsw.knn(tsw.Dataset(X), Q, 3, "dtw", r)
            for j in range(len(Q)):
                oi, od, _ = port.knn(Q[j], oracle.Dataset(X), 3, "dtw", r)
                assert_knn_equal(gi[j], gd[j], oi, od, f"{variant} d={d} L={L} r={r} q{j}")


@pytest.mark.parametrize("variant", ["tiled", "generic"])
def test_dtw_tiled_large_d(tsw, port, variant, monkeypatch):
    """The tiled-cost large-d path (kernels_dtwt.cu, d >= 5, r <= 31) against the oracle and the
    generic kernel: tiny L (tiles reaching into both guard tiles), L not a multiple of 4 or 32,
    both band parities, r = 0 and r = 31 (the widest band of one warp), thresholds that abandon
    in the first and in later cost phases, and the k-NN pipeline with the cumulative bound."""
    import oracle

    if variant == "generic":
        monkeypatch.setenv("TSW_DTW_GENERIC", "1")
    rng = np.random.default_rng(21)
    for d, L, r in ((5, 1, 0), (6, 2, 1), (5, 3, 2), (5, 37, 5), (7, 64, 31), (16, 256, 26),
                    (16, 130, 13), (24, 100, 30), (16, 50, 0), (9, 300, 12), (16, 45, 44)):
        X = walks(rng, 40, L, d)
        q = walks(rng, 1, L, d)[0]
        st = tsw.Store(X)
        ex, val = tsw.dist_all(st, q, "dtw", r)
        ref = port.dtw_all(q, oracle.Dataset(X), r)
        assert ex.all() and np.array_equal(val.view(np.uint64), ref.view(np.uint64)), (d, L, r)
        for eps in (float(np.quantile(ref, 0.05)), float(np.median(ref)), float(ref.min()) * 0.5):
            ex2, val2 = tsw.dist_all(st, q, "dtw", r, eps)
            for i in range(len(X)):
                oe, ov = port.dtw_early_abandon(q, X[i], r, eps)
                assert ex2[i] == oe and val2[i] == ov, (d, L, r, eps, i, ex2[i], val2[i], oe, ov)
        Q = np.concatenate([q[None], X[3:4] + 1e-3, walks(rng, 2, L, d)])
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, 3, "dtw", r)
        for j in range(len(Q)):
            oi, od, _ = port.knn(Q[j], oracle.Dataset(X), 3, "dtw", r)
            assert_knn_equal(gi[j], gd[j], oi, od, f"{variant} d={d} L={L} r={r} q{j}")
            assert gc[j][0] == 40 and gc[j][1] + gc[j][2] + gc[j][3] == 40


def test_dtw_spec_kats(tsw):
    # s=((0),(0)), t=((1),(1)), r=1 -> 2 ; s=t -> 0
    ex, val = tsw.dist_all(tsw.Store(np.ones((1, 2, 1))), np.zeros((2, 1)), "dtw", 1)
    assert ex[0] and val[0] == 2.0
    ex, val = tsw.dist_all(tsw.Store(np.arange(5.0).reshape(1, 5, 1)), np.arange(5.0).reshape(5, 1), "dtw", 2)
    assert val[0] == 0.0
    # eps = 0 with positive first-cell cost -> Exceeds(0)
    ex, val = tsw.dist_all(tsw.Store(np.ones((1, 2, 1))), np.zeros((2, 1)), "dtw", 1, 0.0)
    assert not ex[0] and val[0] == 0.0


# ---- K5 DK DP ----------------------------------------------------------------------------
@pytest.mark.parametrize("N,L,d", [(200, 1, 1), (200, 2, 2), (300, 16, 2), (300, 33, 3),
                                   (200, 64, 1), (200, 128, 2), (100, 256, 16), (20, 1024, 3),
                                   (50, 70, 5)])
def test_dk_all_bit_exact(tsw, port, N, L, d):
    import oracle

    X = walks(RNG, N, L, d)
    q = walks(RNG, 1, L, d)[0]
    st = tsw.Store(X)
    ex, val = tsw.dist_all(st, q, "dk")
    ref = port.dk_all(q, oracle.Dataset(X))
    assert ex.all()
    assert np.array_equal(val.view(np.uint64), ref.view(np.uint64))
    for eps in (float(np.quantile(ref, 0.1)), float(np.median(ref)), 0.0):
        ex2, val2 = tsw.dist_all(st, q, "dk", 0, eps)
        for i in range(N):
            oe, ov = port.sparse_dk(q, X[i], eps)
            assert ex2[i] == oe and val2[i] == ov, (eps, i, ex2[i], val2[i], oe, ov)


@pytest.mark.parametrize("L,d,m", [(200, 2, 200), (300, 3, 150), (130, 1, 260), (257, 2, 129)])
def test_dk_thresholds_multi_strip(tsw, port, L, d, m):
    """Thresholded DK over queries spanning several 64/128-row strips, at 12 thresholds: the
    strip sweep restarts at live boundary cells after dead cuts (a live boundary cell at the
    cut column still reaches the next column diagonally); Exact/Exceeds and values must equal
    sparse_dk (dogkeeper.cpp:227-233) for every candidate."""
    rng = np.random.default_rng(L * 7 + d)
    X = walks(rng, 120, L, d) * 0.3
    q = walks(rng, 1, m, d)[0] * 0.3
    X[5, : min(L, m)] = q[: min(L, m)] + 0.05 * rng.standard_normal((min(L, m), d))
    st = tsw.Store(X)
    ex, full = tsw.dist_all(st, q, "dk")
    assert ex.all()
    for eps in np.quantile(full, np.linspace(0.0, 0.9, 12)):
        ex2, val2 = tsw.dist_all(st, q, "dk", 0, float(eps))
        for i in range(len(X)):
            oe, ov = port.sparse_dk(q, X[i], float(eps))
            assert ex2[i] == oe and val2[i] == ov, (eps, i, ex2[i], val2[i], oe, ov)


def test_dk_ragged_lengths(tsw, port):
    series = [RNG.standard_normal((int(RNG.integers(1, 90)), 3)).cumsum(0) for _ in range(150)]
    q = RNG.standard_normal((57, 3)).cumsum(0)
    ex, val = tsw.dist_all(tsw.Store(series), q, "dk")
    ref = np.array([port.dk_full(q, s) for s in series])
    assert ex.all() and np.array_equal(val.view(np.uint64), ref.view(np.uint64))


def test_dk_spec_kats(tsw):
    # s=((0),(0)), t=((1),(1)) -> 1 ; s=((0),(10),(0)), t=((0),(0)) -> 10
    _, v = tsw.dist_all(tsw.Store(np.ones((1, 2, 1))), np.zeros((2, 1)), "dk")
    assert v[0] == 1.0
    _, v = tsw.dist_all(tsw.Store([np.zeros((2, 1))]), np.array([[0.0], [10.0], [0.0]]), "dk")
    assert v[0] == 10.0


# ---- k-NN drivers vs the reference (acceptance criterion 8) -----------------
def _check_counters(c, n, metric):
    if metric == "dtw":
        assert c[0] == n and c[1] + c[2] + c[3] == n, c
    else:
        assert c[4] == seed_sample(n) and c[2] + c[3] == n, c


def test_counters_device_counted_no_pruning(tsw):
    """k >= n: the threshold never drops below +inf, so nothing can be pruned or abandoned --
    every candidate must be counted by the DP as full_dp (device counters, not complements)."""
    X = RNG.standard_normal((37, 24, 2)).cumsum(1)
    qs = RNG.standard_normal((3, 24, 2)).cumsum(1)
    ds = tsw.Store(X)
    for metric in ("dtw", "dk"):
        _, _, ctr = tsw.knn(ds, qs, 40, metric, 3)
        for c in ctr:
            if metric == "dtw":
                assert list(c) == [37, 0, 37, 0, 0], c
            else:
                assert list(c) == [0, 0, 37, 0, 37], c


def test_counters_prune_and_abandon(tsw):
    """1-NN where one candidate equals the query: after it is found everything else is
    pruned by a bound or abandoned; the device counts must add up to n (checked by the
    library too) and show real pruning."""
    X = RNG.standard_normal((3000, 64, 3)).cumsum(1)
    q = X[1234].copy()
    ds = tsw.Store(X)
    _, _, c = tsw.knn(ds, q[None], 1, "dtw", 6)
    c = c[0]
    assert c[0] == 3000 and c[1] + c[2] + c[3] == 3000 and c[1] > 2000 and c[2] >= 1, c
    _, _, c = tsw.knn(ds, q[None], 1, "dk", 0)
    c = c[0]
    assert c[2] + c[3] == 3000 and c[2] >= 1 and c[3] > 2000 and c[4] == seed_sample(3000, 64, 3, 1, nq=1), c


def test_knn_random_datasets(tsw, best_oracle):
    import oracle

    rng = np.random.default_rng(8)
    for trial in range(100):
        n = int(rng.integers(1, 200))
        L = int(rng.integers(1, 64))
        d = int(rng.integers(1, 5))
        r = int(rng.integers(0, max(1, L // 3) + 1))
        k = int(rng.integers(1, 12))
        X = walks(rng, n, L, d)
        Q = walks(rng, 3, L, d)
        if trial % 10 == 0:
            Q[0] = X[int(rng.integers(0, n))]  # query in data: self-match at distance 0
        ds = tsw.Dataset(X)
        ods = oracle.Dataset(X)
        for metric in ("dtw", "dk"):
            gi, gd, gc = tsw.knn(ds, Q, k, metric, r)
            for q in range(len(Q)):
                oi, od, _ = best_oracle.knn(Q[q], ods, k, metric, r)
                assert_knn_equal(gi[q], gd[q], oi, od, f"trial {trial} {metric} q{q}")
                _check_counters(gc[q], n, metric)


@pytest.mark.parametrize("lb2", ["0", "1"])
def test_knn_values_beyond_fp32_range(tsw, best_oracle, lb2, monkeypatch):
    """The reference accepts any finite double (timeseries.cpp:16-21).  Values beyond FLT_MAX
    (1e39) and values whose squared differences overflow fp64 (1e200: DTW/DK costs of +inf)
    must give the reference's neighbours: the fp32 LB shadow saturates instead of producing
    +inf terms that would prune true neighbours."""
    import oracle

    monkeypatch.setenv("TSW_LB2", lb2)
    rng = np.random.default_rng(41)
    for scale_db, scale_q in ((1e39, 1e39), (1e39, 1.0), (1.0, 1e39), (1e200, 1e200)):
        n, L, d, r, k = 400, 40, 3, 5, 3
        X = walks(rng, n, L, d)
        X[::3] *= scale_db  # a third of the store beyond fp32 range
        Q = walks(rng, 4, L, d) * scale_q
        Q[1] = X[9] * (1 + 1e-9)
        Q[2] = X[10]
        ds = tsw.Dataset(X)
        ods = oracle.Dataset(X)
        # DK at 1e200 (point distances of +inf) is undefined behaviour in the reference: its
        # greedy walk (dogkeeper.cpp:60-84) steps past the last row when every move costs +inf
        # (strict < never prefers the in-range move) and reads out of bounds -- the reference
        # and its C restatement crash there, so there is nothing to compare against
        for metric in (("dtw",) if scale_db > 1e150 else ("dtw", "dk")):
            gi, gd, gc = tsw.knn(ds, Q, k, metric, r)
            for q in range(len(Q)):
                oi, od, _ = best_oracle.knn(Q[q], ods, k, metric, r)
                keep = gi[q] != tsw.NO_NEIGHBOR  # short rows: the reference's KBest ends short
                assert_knn_equal(gi[q][keep], gd[q][keep], oi, od, f"{scale_db} {scale_q} {metric} q{q}")
                rep = (tsw.knn_dtw(Q[q], ds, k, r) if metric == "dtw" else tsw.knn_dk(Q[q], ds, k))
                assert [nb.index for nb in rep.neighbors] == [int(i) for i in oi]
                _check_counters(gc[q], n, metric)


@pytest.mark.parametrize("lb2", ["0", "1"])
def test_knn_reverse_bound_modes(tsw, best_oracle, lb2, monkeypatch):
    """The fused forward + reverse LB_Box pass (TSW_LB2=1: query points against the candidate
    envelope) and the forward-only pass give the reference's neighbours on the same inputs:
    ragged tails (L not a multiple of 32), d = 1..5, LB block-sum rows on and off (L <= 256 /
    longer), narrow and wide bands."""
    import oracle

    monkeypatch.setenv("TSW_LB2", lb2)
    rng = np.random.default_rng(31)
    for n, L, d, r, k in ((150, 20, 1, 3, 2), (300, 45, 3, 6, 1), (200, 97, 2, 20, 4),
                          (120, 130, 4, 40, 3), (80, 300, 3, 33, 2), (60, 64, 5, 10, 5)):
        X = walks(rng, n, L, d)
        Q = walks(rng, 4, L, d)
        Q[1] = X[7] + 1e-3 * rng.standard_normal((L, d))
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
        ods = oracle.Dataset(X)
        for q in range(len(Q)):
            oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
            assert_knn_equal(gi[q], gd[q], oi, od, f"lb2={lb2} n={n} L={L} d={d} r={r} q{q}")
            _check_counters(gc[q], n, "dtw")


def test_knn_ties_and_duplicates(tsw, best_oracle):
    import oracle

    base = walks(RNG, 20, 24, 2)
    X = np.concatenate([base, base, base[::-1]])  # exact duplicates -> equal distances
    q = base[3] + 0.01
    for metric in ("dtw", "dk"):
        for k in (1, 2, 3, 7, 40, 60):
            gi, gd, _ = tsw.knn(tsw.Dataset(X), q[None], k, metric, 4)
            oi, od, _ = best_oracle.knn(q, oracle.Dataset(X), k, metric, 4)
            assert_knn_equal(gi[0], gd[0], oi, od, f"{metric} k={k}")


def test_knn_k_larger_than_kmax_and_n(tsw, best_oracle):
    import oracle

    X = walks(RNG, 150, 20, 2)
    q = walks(RNG, 1, 20, 2)[0]
    for metric in ("dtw", "dk"):
        for k in (65, 100, 150, 1000):
            gi, gd, gc = tsw.knn(tsw.Dataset(X), q[None], k, metric, 3)
            oi, od, _ = best_oracle.knn(q, oracle.Dataset(X), k, metric, 3)
            assert_knn_equal(gi[0], gd[0], oi, od, f"{metric} k={k}")
            _check_counters(gc[0], 150, metric)


def test_knn_constant_and_degenerate(tsw, best_oracle):
    import oracle

    X = np.zeros((30, 10, 2))
    X[5] += 1.0
    q = np.zeros((10, 2))
    for metric in ("dtw", "dk"):
        gi, gd, _ = tsw.knn(tsw.Dataset(X), q[None], 4, metric, 2)
        oi, od, _ = best_oracle.knn(q, oracle.Dataset(X), 4, metric, 2)
        assert_knn_equal(gi[0], gd[0], oi, od, metric)


def test_knn_dk_ragged(tsw, best_oracle):
    import oracle

    series = [RNG.standard_normal((int(RNG.integers(1, 80)), 2)).cumsum(0) for _ in range(120)]
    for k in (1, 5):
        q = RNG.standard_normal((40, 2)).cumsum(0)
        rep = tsw.knn_dk(q, tsw.Dataset(series), k)
        oi, od, _ = best_oracle.knn(q, oracle.Dataset(series), k, "dk")
        assert_knn_equal([nb.index for nb in rep.neighbors], [nb.distance for nb in rep.neighbors], oi, od)


def test_errors_mirror_reference(tsw):
    X = walks(RNG, 10, 12, 2)
    ds = tsw.Dataset(X)
    with pytest.raises(ValueError, match="k must be positive"):
        tsw.knn_dtw(X[0], ds, 0, 2)
    with pytest.raises(ValueError, match="query dim"):
        tsw.knn_dk(np.zeros((12, 3)), ds, 1)
    with pytest.raises(ValueError, match="length differs"):
        tsw.knn_dtw(np.zeros((11, 2)), ds, 1, 2)
    with pytest.raises(ValueError, match="eps must be nonnegative"):
        tsw.epsnn_dk(X[0], ds, -1.0)
    with pytest.raises(tsw.ValidationError):
        tsw.Store(np.full((2, 3, 1), np.nan))


def test_epsnn_dk(tsw, best_oracle):
    import oracle

    X = walks(RNG, 300, 30, 3)
    q = walks(RNG, 1, 30, 3)[0]
    ods = oracle.Dataset(X)
    dks = np.array([best_oracle.dk_full(q, x) for x in X])
    for eps in (0.0, float(np.quantile(dks, 0.05)), float(np.median(dks)), float("inf")):
        rep = tsw.epsnn_dk(q, tsw.Dataset(X), eps)
        oi, od, _ = best_oracle.epsnn_dk(q, ods, eps)
        assert_knn_equal([nb.index for nb in rep.neighbors], [nb.distance for nb in rep.neighbors], oi, od)
        assert rep.counters.full_dp + rep.counters.early_abandoned == 300


def test_plan_reuse_and_device_queries(tsw, best_oracle):
    import oracle
    import torch

    X = walks(RNG, 500, 64, 3)
    Q = walks(RNG, 6, 64, 3)
    ds = tsw.Dataset(X)
    plan = tsw.Plan(ds, 8, 64, "dtw", 6, 3)
    plan.set_queries(Q)
    plan.execute()
    a = plan.fetch()
    dq = torch.from_numpy(Q).cuda()
    stream = torch.cuda.current_stream()
    plan.set_queries_device(dq.data_ptr(), 6, stream.cuda_stream)
    plan.execute(stream.cuda_stream)
    b = plan.fetch(stream.cuda_stream)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for q in range(6):
        oi, od, _ = best_oracle.knn(Q[q], oracle.Dataset(X), 3, "dtw", 6)
        assert_knn_equal(a[0][q], a[1][q], oi, od)


def test_plan_cuda_graph_matches_eager(tsw):
    X = walks(RNG, 700, 64, 3)
    Q = walks(RNG, 9, 64, 3)
    for metric in ("dtw", "dk"):
        eager = tsw.Plan(tsw.Dataset(X), 9, 64, metric, 6, 4)
        eager.set_queries(Q)
        eager.execute()
        a = eager.fetch()
        g = tsw.Plan(tsw.Dataset(X), 9, 64, metric, 6, 4)
        g.set_graph(True)
        for _ in range(3):  # warm execute, capture, replay
            g.set_queries(Q)
            g.execute()
            b = g.fetch()
            # neighbours are deterministic; counters depend on the threshold schedule (only
            # their conservation identity is a contract)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            for c in b[2]:
                assert c[2] + c[3] + (c[1] if metric == "dtw" else 0) == 700


@pytest.mark.parametrize("env", ["1", "0"])
def test_knn_lb_envelope_paths(tsw, best_oracle, env, monkeypatch):
    """K2 with the query envelopes staged in shared memory (lb_env_kernel, TSW_LB_ENV=1, the
    default for L*d <= 768) and the L1 tile kernel (TSW_LB_ENV=0) give the reference's
    neighbours: query counts that are not multiples of the 8-query block, candidate counts that
    are not multiples of the 4-candidate group, lengths that are not multiples of 32, block-sum
    rows on (L <= 256), and a store long enough for several candidate chunks per block."""
    import oracle

    monkeypatch.setenv("TSW_LB_ENV", env)
    rng = np.random.default_rng(77)
    for n, L, d, r, k, nq in ((1001, 40, 3, 4, 1, 9), (333, 128, 3, 13, 3, 17),
                              (2050, 96, 2, 9, 2, 5), (517, 190, 4, 19, 1, 12)):
        X = walks(rng, n, L, d)
        Q = walks(rng, nq, L, d)
        Q[2] = X[11] + 1e-3 * rng.standard_normal((L, d))
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
        ods = oracle.Dataset(X)
        for q in range(nq):
            oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
            assert_knn_equal(gi[q], gd[q], oi, od, f"env={env} n={n} L={L} d={d} r={r} q{q}")
            _check_counters(gc[q], n, "dtw")


def test_knn_lb_envelope_many_query_blocks(tsw, best_oracle):
    """More 8-query blocks (313) than resident LB blocks (2 per SM): the blocks of the
    shared-memory-envelope K2 then change query block from one work item to the next and
    re-stage the envelopes; sampled queries equal the reference's neighbours."""
    import oracle

    rng = np.random.default_rng(2500)
    n, L, d, r, k, nq = 300, 32, 2, 3, 2, 2500
    X = walks(rng, n, L, d)
    Q = walks(rng, nq, L, d)
    Q[1234] = X[42] + 1e-3 * rng.standard_normal((L, d))
    gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
    ods = oracle.Dataset(X)
    for q in (0, 1, 7, 8, 1234, 2367, 2368, 2499):
        oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
        assert_knn_equal(gi[q], gd[q], oi, od, f"q{q}")
        _check_counters(gc[q], n, "dtw")


def test_concurrent_knn_calls_on_one_store(tsw):
    """tsw_knn calls on one store from several host threads run concurrently (pooled plans,
    no store-wide lock held during execution) and give the sequential answers."""
    import threading

    rng = np.random.default_rng(77)
    X = walks(rng, 4000, 96, 3)
    ds = tsw.Store(X)
    Qs = [walks(rng, 5, 96, 3) for _ in range(6)]
    want = [tsw.knn(ds, Q, 3, "dtw" if i % 2 == 0 else "dk", 9) for i, Q in enumerate(Qs)]
    got = [None] * len(Qs)
    errs = []

    def run(i):
        try:
            for _ in range(3):
                got[i] = tsw.knn(ds, Qs[i], 3, "dtw" if i % 2 == 0 else "dk", 9)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(Qs))]
    for t_ in th:
        t_.start()
    for t_ in th:
        t_.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert np.array_equal(w[0], g[0]) and np.array_equal(w[1], g[1])


@pytest.mark.parametrize("limit", [None, "2048"])
def test_long_series_beyond_shared_memory(tsw, best_oracle, limit, monkeypatch):
    """Series long enough that the DP kernels' per-block arrays (DTW prefix bounds, DK boundary
    rows) exceed the shared-memory limit run with those arrays in global scratch and still give
    the reference's answers; TSW_SMEM_LIMIT forces the same spill mode at short lengths."""
    import oracle

    if limit:
        monkeypatch.setenv("TSW_SMEM_LIMIT", limit)
        cases = [("dtw", 200, 300, 3, 20), ("dtw", 120, 180, 2, 70), ("dtw", 60, 200, 16, 20),
                 ("dk", 150, 260, 2, 0)]
    else:
        cases = [("dtw", 24, 4500, 3, 40), ("dtw", 16, 4200, 2, 300), ("dk", 10, 8000, 2, 0)]
    rng = np.random.default_rng(5)
    for metric, n, L, d, r in cases:
        X = walks(rng, n, L, d)
        Q = walks(rng, 2, L, d)
        Q[1] = X[3] + 0.01 * rng.standard_normal((L, d))
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, 2, metric, r)
        ods = oracle.Dataset(X)
        for q in range(len(Q)):
            oi, od, _ = best_oracle.knn(Q[q], ods, 2, metric, r)
            assert_knn_equal(gi[q], gd[q], oi, od, f"{metric} L={L} r={r} q{q}")
            _check_counters(gc[q], n, metric)


@pytest.mark.parametrize("revcb,noidle", [("1", None), ("0", None), ("1", "1")])
def test_dtw_fast_path_variants(tsw, best_oracle, revcb, noidle, monkeypatch):
    """The DTW fast path with and without the reverse cumulative abandon bound (query rows
    ahead against the candidate envelope, r >= 32) and with / without the +inf idle lanes:
    the reference's neighbours and distances on wide bands, L above and below 256, d = 1..4,
    1 to 6 queries (the 1-3 query plans skip the reverse LB pass but keep the DP bound)."""
    import oracle

    monkeypatch.setenv("TSW_REVCB", revcb)
    if noidle:
        monkeypatch.setenv("TSW_DTW4_NOIDLE", noidle)
    rng = np.random.default_rng(91)
    for n, L, d, r, k, nq in ((300, 120, 3, 32, 3, 6), (200, 300, 2, 40, 2, 2), (150, 97, 1, 35, 4, 5),
                              (120, 520, 4, 51, 1, 1), (250, 64, 3, 13, 2, 4), (180, 200, 2, 26, 3, 4)):
        X = walks(rng, n, L, d)
        Q = walks(rng, nq, L, d)
        Q[0] = X[5] + 1e-3 * rng.standard_normal((L, d))
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
        ods = oracle.Dataset(X)
        for q in range(nq):
            oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
            assert_knn_equal(gi[q], gd[q], oi, od, f"n={n} L={L} d={d} r={r} q{q}")
            _check_counters(gc[q], n, "dtw")


def test_lb_box_exact_and_pruning_power_match_reference(tsw, best_oracle):
    """tsw_lb_box_exact_all is the reference's fp64 lb_box bit for bit, and pruning_power
    replays the reference's 1-NN scan schedule exactly: its pruned count equals the sum of the
    reference knn_dtw's lb_pruned counters (deterministic, unlike this engine's own counters)."""
    import oracle

    rng = np.random.default_rng(12)
    for n, L, d, r in ((700, 60, 3, 6), (300, 128, 2, 13), (257, 33, 1, 0)):
        X = walks(rng, n, L, d)
        Q = walks(rng, 5, L, d)
        Q[2] = X[100]  # self-match: distance 0 found mid-scan
        st = tsw.Store(X)
        for q in Q[:2]:
            lb = tsw.lb_box_exact_all(st, q, r)
            ref = np.array([best_oracle.lb_box(X[i], q, r) for i in range(n)])
            assert np.array_equal(lb.view(np.uint64), ref.view(np.uint64))
        ds = tsw.Dataset(X)
        pp = tsw.pruning_power(tsw.Dataset(list(Q)), ds, r)
        ods = oracle.Dataset(X)
        pruned = sum(int(best_oracle.knn(q, ods, 1, "dtw", r)[2][1]) for q in Q)
        assert pp == pruned / (len(Q) * n), (pp, pruned)


@pytest.mark.parametrize("stages", ["1", "2"])
def test_staged_dtw_execution(tsw, best_oracle, stages, monkeypatch):
    """Staged DTW execution (the first quarter of the candidates bounded and DP'd first, the
    rest against the stage-1 threshold; default for n >= 96k) gives the reference's neighbours
    through every LB pass variant: shared-memory envelopes (short series), the L1 tile pass,
    the fused reverse pass (r >= 32) and the 1-3 query pass."""
    import oracle

    monkeypatch.setenv("TSW_STAGES", stages)
    rng = np.random.default_rng(404)
    for n, L, d, r, k, nq in ((2001, 64, 3, 6, 3, 9), (1500, 300, 2, 40, 2, 6), (900, 96, 6, 9, 1, 5),
                              (1203, 128, 3, 13, 4, 2), (640, 200, 3, 51, 10, 4)):
        X = walks(rng, n, L, d)
        Q = walks(rng, nq, L, d)
        Q[0] = X[n - 7] + 1e-3 * rng.standard_normal((L, d))  # a neighbour in stage 2
        Q[-1] = X[3] + 1e-3 * rng.standard_normal((L, d))     # ... and one in stage 1
        gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
        ods = oracle.Dataset(X)
        for q in range(nq):
            oi, od, _ = best_oracle.knn(Q[q], ods, k, "dtw", r)
            assert_knn_equal(gi[q], gd[q], oi, od, f"stages={stages} n={n} L={L} d={d} r={r} q{q}")
            _check_counters(gc[q], n, "dtw")
