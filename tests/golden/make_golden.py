"""Generate the golden parity fixtures from the REFERENCE itself (oracle/_ref, compiled from
/root/reference/proj/core/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

Writes tests/golden/reference_vectors.json: small seeded datasets with the reference's own
outputs for every hot-path function (knn_dtw, knn_dk incl. counters, epsnn_dk, dtw_banded,
dtw_early_abandon, dk_full, sparse_dk, gdk, lb_box, envelope, znormalize).  Doubles are stored
as float.hex() strings so the fixtures are bit-exact.  /root/reference does not exist on the GPU
box; the committed JSON travels instead.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

SEED = 1811_11076


def hx(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def walks(rng, n, L, d):
    x = rng.standard_normal((n, L, d)).cumsum(1)
    return x


def main():
    R = oracle.ref()
    rng = np.random.default_rng(SEED)
    cases = []
    shapes = [  # (n, L, d, r, ks, nq, ragged)
        (40, 16, 1, 2, [1, 3], 2, False),
        (64, 24, 2, 3, [1, 5], 2, False),
        (50, 32, 3, 4, [1, 4, 50], 2, False),
        (30, 20, 16, 2, [1, 2], 2, False),
        (25, 12, 2, 0, [1, 30], 2, False),
        (45, 1, 2, 0, [1, 3], 1, False),
        (36, 0, 3, 0, [1, 6], 2, True),   # ragged lengths (DK only)
    ]
    for ci, (n, L, d, r, ks, nq, ragged) in enumerate(shapes):
        if ragged:
            series = [rng.standard_normal((int(rng.integers(1, 30)), d)).cumsum(0) for _ in range(n)]
            qlen = 17
            queries = [rng.standard_normal((qlen, d)).cumsum(0) for _ in range(nq)]
        else:
            X = walks(rng, n, L, d)
            if ci == 2:
                X[7] = X[3]  # exact duplicate: tie broken by lower index
            series = list(X)
            queries = list(walks(rng, nq, L, d))
            if ci == 1:
                queries[0] = X[11].copy()  # self-match at distance 0
        ds = oracle.Dataset(series)
        case = {"name": f"case{ci}", "d": d, "r": r, "ragged": ragged,
                "series": [hx(s) for s in series], "lengths": [len(s) for s in series],
                "queries": [hx(q) for q in queries], "qlen": len(queries[0]), "knn": [],
                "pair": []}
        for qi, q in enumerate(queries):
            for metric in (["dk"] if ragged else ["dtw", "dk"]):
                for k in ks:
                    idx, dist, ctr = R.knn(q, ds, k, metric, r)
                    case["knn"].append({"q": qi, "metric": metric, "k": k,
                                        "index": [int(i) for i in idx], "distance": hx(dist),
                                        "counters": [int(c) for c in ctr]})
            dks = [R.dk_full(q, s) for s in series]
            eps = float(np.median(dks))
            ei, ed, _ = R.epsnn_dk(q, ds, eps)
            case.setdefault("epsnn", []).append({"q": qi, "eps": float(eps).hex(),
                                                 "index": [int(i) for i in ei], "distance": hx(ed)})
        # per-pair primitives against the first query
        q = queries[0]
        for si, s in enumerate(series[:12]):
            ent = {"i": si, "dk_full": float(R.dk_full(q, s)).hex(),
                   "gdk": float(R.gdk(q, s)).hex()}
            ex, v = R.sparse_dk(q, s, float(R.dk_full(q, s)) * 0.999)
            ent["sparse_dk_below"] = [ex, float(v).hex()]
            if not ragged:
                ent["dtw_banded"] = float(R.dtw_banded(q, s, r)).hex()
                ex, v = R.dtw_early_abandon(q, s, r, float(R.dtw_banded(q, s, r)))
                ent["dtw_early_abandon_at_d"] = [ex, float(v).hex()]
                ent["lb_box"] = float(R.lb_box(s, q, r)).hex()
            case["pair"].append(ent)
        if not ragged:
            lo, hi = R.envelope(q, r)
            case["envelope_q0"] = {"lo": hx(lo), "hi": hx(hi)}
            case["znormalize_q0"] = hx(R.znormalize(q))
        cases.append(case)
    out = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libtswarp_ref.so "
           "(reference sources compiled with -O3 -DNDEBUG -ffp-contract=off)", "seed": SEED,
           "cases": cases}
    path = os.path.join(HERE, "reference_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB, {len(cases)} cases)")


def main_sub():
    """Subsequence DK fixtures: knn_dk_sub, sparse_dk_sub, sub_search_dk and
    gdk_sub from the reference, on short queries inside longer (and ragged) haystacks."""
    R = oracle.ref()
    rng = np.random.default_rng(SEED + 2)
    cases = []
    shapes = [  # (n, haystack length range, d, query lengths, ks)
        (40, (30, 31), 1, [6, 12], [1, 3]),
        (50, (20, 60), 2, [5, 17], [1, 5, 50]),
        (30, (8, 40), 3, [9, 45], [1, 4]),
        (20, (24, 25), 16, [7], [1, 2]),
    ]
    for ci, (n, (lmin, lmax), d, qlens, ks) in enumerate(shapes):
        series = [rng.standard_normal((int(rng.integers(lmin, lmax)), d)).cumsum(0) for _ in range(n)]
        queries = [rng.standard_normal((m, d)).cumsum(0) for m in qlens]
        if ci == 1:
            # a query cut out of a haystack: an exact subsequence match at distance 0
            queries[0] = series[9][3:8].copy()
            series[21] = series[9].copy()  # duplicate haystack: tie broken by lower index
        ds = oracle.Dataset(series)
        case = {"name": f"sub{ci}", "d": d, "series": [hx(x) for x in series],
                "queries": [hx(q) for q in queries], "qlens": qlens, "knn": [], "pair": []}
        for qi, q in enumerate(queries):
            for k in ks:
                idx, dist, ctr = R.knn(q, ds, k, "dk_sub")
                case["knn"].append({"q": qi, "k": k, "index": [int(i) for i in idx],
                                    "distance": hx(dist), "counters": [int(c) for c in ctr]})
            for si, x in enumerate(series[:10]):
                full = R.sparse_dk_sub(q, x, float("inf"))
                ent = {"q": qi, "i": si, "sub_inf": [full[0].hex(), full[1]],
                       "gdk_sub": [R.gdk_sub(q, x)[0].hex(), R.gdk_sub(q, x)[1]]}
                below = R.sparse_dk_sub(q, x, full[0] * 0.999)
                ent["sub_below"] = None if below is None else [below[0].hex(), below[1]]
                at = R.sub_search_dk(q, x, full[0])
                ent["search_at"] = None if at is None else [at[0].hex(), at[1]]
                case["pair"].append(ent)
        cases.append(case)
    out = {"generator": "tests/golden/make_golden.py (main_sub)",
           "reference": "oracle/_ref/libtswarp_ref.so", "seed": SEED + 2, "cases": cases}
    path = os.path.join(HERE, "reference_sub_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB, {len(cases)} cases)")


IO_DOCS = [  # (name, document bytes): valid files, number/strings edge cases, every error path
    ("basic", b'{"dim": 2, "meta": {"src": "unit", "a": "b"}, "series": [{"label": "A", "points": [[1, 2], [3.5, -4e-3]]}, {"label": "B", "points": [[0.1, 0.2]]}]}'),
    ("unlabeled_ragged", b'{"dim":1,"series":[{"points":[[1],[2],[3]]},{"points":[[4]]}]}'),
    ("no_meta_ws", b' \r\n\t{ "series" : [ { "points" : [ [ 7 ] ] } ] , "dim" : 1 } \n'),
    ("bom", b'\xef\xbb\xbf{"dim":1,"series":[{"points":[[1]]}]}'),
    ("numbers", b'{"dim":1,"series":[{"points":[[-0],[-0.0],[0.1],[1e400],[1E5],[123456789012345678901234567890],[-9223372036854775809],[18446744073709551615],[18446744073709551616],[9007199254740993],[1.7976931348623157e308],[4.9e-324],[1e-400],[2.2250738585072011e-308],[0.30000000000000004],[-1.5e+2]]}]}'),
    ("numbers_finite", b'{"dim":1,"series":[{"points":[[-0],[-0.0],[0.1],[1E5],[123456789012345678901234567890],[-9223372036854775809],[18446744073709551615],[18446744073709551616],[9007199254740993],[1.7976931348623157e308],[4.9e-324],[1e-400],[2.2250738585072011e-308],[0.30000000000000004],[-1.5e+2]]}]}'),
    ("strings", b'{"dim":1,"meta":{"k\\u00e9y":"v\\n\\t\\"q\\"","emoji":"\\ud83d\\ude00","raw":"\xc3\xa9\xe2\x82\xac"},"series":[{"label":"\\u0041\\/b","points":[[1]]}]}'),
    ("dup_keys", b'{"dim":3,"dim":1,"series":[{"points":[[1]]}],"meta":{"a":"1","a":"2"}}'),
    ("extra_keys", b'{"dim":1,"x":[1,{"y":null}],"series":[{"points":[[1]],"other":true}]}'),
    ("empty", b''),
    ("not_object", b'[1,2]'),
    ("missing_series", b'{"dim":1}'),
    ("missing_dim", b'{"series":[{"points":[[1]]}]}'),
    ("dim_zero", b'{"dim":0,"series":[{"points":[[1]]}]}'),
    ("dim_negative", b'{"dim":-1,"series":[{"points":[[1]]}]}'),
    ("dim_float", b'{"dim":1.0,"series":[{"points":[[1]]}]}'),
    ("dim_string", b'{"dim":"1","series":[{"points":[[1]]}]}'),
    ("meta_not_object", b'{"dim":1,"meta":[],"series":[{"points":[[1]]}]}'),
    ("meta_value", b'{"dim":1,"meta":{"a":"x","b":2},"series":[{"points":[[1]]}]}'),
    ("series_empty", b'{"dim":1,"series":[]}'),
    ("series_not_array", b'{"dim":1,"series":{"points":[[1]]}}'),
    ("series_item", b'{"dim":1,"series":[{"points":[[1]]},[1]]}'),
    ("series_no_points", b'{"dim":1,"series":[{"label":"a"}]}'),
    ("label_type", b'{"dim":1,"series":[{"label":1,"points":[[1]]}]}'),
    ("points_empty", b'{"dim":1,"series":[{"points":[]}]}'),
    ("points_type", b'{"dim":1,"series":[{"points":5}]}'),
    ("point_type", b'{"dim":1,"series":[{"points":[[1],2]}]}'),
    ("point_size", b'{"dim":2,"series":[{"points":[[1,2],[3]]}]}'),
    ("component_string", b'{"dim":2,"series":[{"points":[[1,"2"]]}]}'),
    ("component_null", b'{"dim":1,"series":[{"points":[[null]]}]}'),
    ("component_bool", b'{"dim":1,"series":[{"points":[[true]]}]}'),
    ("nonfinite", b'{"dim":2,"series":[{"points":[[1,2]]},{"points":[[1,2],[3,-1e999]]}]}'),
    ("labels_mixed", b'{"dim":1,"series":[{"label":"a","points":[[1]]},{"points":[[2]]}]}'),
    ("labels_mixed2", b'{"dim":1,"series":[{"points":[[1]]},{"label":"b","points":[[2]]}]}'),
    ("size_before_label_mix", b'{"dim":1,"series":[{"label":"a","points":[[1]]},{"points":[[2,3]]}]}'),
    ("trailing_comma", b'{"dim":1,"series":[{"points":[[1],]}]}'),
    ("trailing_garbage", b'{"dim":1,"series":[{"points":[[1]]}]} x'),
    ("two_docs", b'{"dim":1,"series":[{"points":[[1]]}]}{}'),
    ("leading_zero", b'{"dim":1,"series":[{"points":[[01]]}]}'),
    ("plus", b'{"dim":1,"series":[{"points":[[+1]]}]}'),
    ("dot", b'{"dim":1,"series":[{"points":[[.5]]}]}'),
    ("nan", b'{"dim":1,"series":[{"points":[[NaN]]}]}'),
    ("infinity", b'{"dim":1,"series":[{"points":[[Infinity]]}]}'),
    ("frac_missing", b'{"dim":1,"series":[{"points":[[1.]]}]}'),
    ("exp_missing", b'{"dim":1,"series":[{"points":[[1e]]}]}'),
    ("single_quote", b"{'dim':1}"),
    ("control_char", b'{"dim":1,"series":[{"label":"a\tb","points":[[1]]}]}'),
    ("bad_escape", b'{"dim":1,"series":[{"label":"a\\x","points":[[1]]}]}'),
    ("lone_surrogate", b'{"dim":1,"series":[{"label":"\\udc00","points":[[1]]}]}'),
    ("high_surrogate_alone", b'{"dim":1,"series":[{"label":"\\ud800x","points":[[1]]}]}'),
    ("bad_utf8", b'{"dim":1,"series":[{"label":"\xff","points":[[1]]}]}'),
    ("overlong_utf8", b'{"dim":1,"series":[{"label":"\xc0\xaf","points":[[1]]}]}'),
    ("unterminated", b'{"dim":1,"series":[{"points":[[1]]}]'),
    ("bad_literal", b'{"dim":1,"series":[{"points":[[1]]}],"x":tru}'),
]


def main_io():
    """Dataset-file fixtures: every IO_DOCS document through the reference's
    own load_dataset (oracle/_ref/libtswarp_ref_io.so, nlohmann/json 3.11.3), recording the
    exception kind + message (with the file path replaced by {path}) or the loaded dataset."""
    import base64
    import tempfile

    RIO = oracle.ref_io()
    out = []
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "doc.json")
        for name, doc in IO_DOCS:
            with open(path, "wb") as f:
                f.write(doc)
            ent = {"name": name, "doc_b64": base64.b64encode(doc).decode()}
            try:
                vals, lens, d, labels, meta = RIO.load(path)
                ent["ok"] = {"d": d, "values": hx(vals), "lengths": [int(x) for x in lens],
                             "labels": labels, "meta": meta}
            except oracle.RefIOError as e:
                ent["error"] = {"kind": e.kind, "message": e.message.replace(path, "{path}")}
            out.append(ent)
    res = {"generator": "tests/golden/make_golden.py (main_io)",
           "reference": "oracle/_ref/libtswarp_ref_io.so (dataset_io.cpp + nlohmann/json 3.11.3)",
           "cases": out}
    p = os.path.join(HERE, "dataset_io_vectors.json")
    with open(p, "w") as f:
        json.dump(res, f, indent=0)
    print(f"wrote {p} ({len(out)} cases)")


if __name__ == "__main__":
    if "--sub" in sys.argv:
        main_sub()
    elif "--io" in sys.argv:
        main_io()
    else:
        main()
        main_sub()
        main_io()
