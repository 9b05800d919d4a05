"""Dataset files: tswarp::load_dataset / save_dataset (dataset_io.cpp:45-140)
restated in csrc/dataset_io.cpp, checked against the reference's own implementation.

* golden: every document of tests/golden/dataset_io_vectors.json (made by the reference's
  load_dataset built against nlohmann/json 3.11.3, tests/golden/make_golden.py --io): the same
  dataset bit for bit, or the same exception type with the same message (messages authored by
  the reference compared exactly; the JSON library's syntax-error texts only by their
  "<path>: " prefix);
* live (when oracle/_ref/libtswarp_ref_io.so is built): random datasets saved by one side load
  bit-exactly on the other, both directions;
* GPU: a loaded file uploads to a device store whose k-NN answers equal the in-memory ones.
Host parsing needs no GPU; only the last test is marked gpu.
"""
import base64
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def unhex(lst):
    return np.array([float.fromhex(v) for v in lst])


@pytest.fixture(scope="module")
def tsw_host():
    import paper_1811_11076_b200 as t

    t.lib()
    return t


@pytest.fixture(scope="module")
def golden_io():
    with open(os.path.join(HERE, "golden", "dataset_io_vectors.json")) as f:
        return json.load(f)


def _flat(ds):
    sers = [np.asarray(ds.series(i)) for i in range(ds.n)]
    return np.concatenate([s.reshape(-1) for s in sers]), [s.shape[0] for s in sers]


KIND = {"ParseError": "ParseError", "ValidationError": "ValidationError", "IoError": "IoError",
        "runtime_error": "ParseError"}  # the JSON library's out_of_range (number overflow)


def test_load_matches_reference_golden(tsw_host, golden_io, tmp_path):
    t = tsw_host
    path = str(tmp_path / "doc.json")
    for case in golden_io["cases"]:
        with open(path, "wb") as f:
            f.write(base64.b64decode(case["doc_b64"]))
        if "ok" in case:
            ds = t.load_dataset(path)
            exp = case["ok"]
            vals, lens = _flat(ds)
            assert ds.dim == exp["d"], case["name"]
            assert lens == exp["lengths"], case["name"]
            assert np.array_equal(vals.view(np.uint64), unhex(exp["values"]).view(np.uint64)), case["name"]
            assert ds.labels == exp["labels"], case["name"]
            assert ds.meta == exp["meta"], case["name"]
        else:
            err = case["error"]
            with pytest.raises(Exception) as ei:
                t.load_dataset(path)
            assert type(ei.value).__name__ == KIND[err["kind"]], (case["name"], ei.value)
            msg = str(ei.value)
            ref = err["message"].replace("{path}", path)
            if "[json.exception" in ref and "number overflow" not in ref:
                assert msg.startswith(path + ": "), (case["name"], msg)
            elif "number overflow" in ref:
                assert ref.split("] ", 1)[1] in msg, (case["name"], msg, ref)
            else:
                assert msg == ref, (case["name"], msg, ref)


def test_io_errors(tsw_host, tmp_path):
    t = tsw_host
    missing = str(tmp_path / "none.json")
    with pytest.raises(t.IoError, match="cannot open .* for reading"):
        t.load_dataset(missing)
    ds = t.Dataset(np.zeros((1, 2, 1)))
    with pytest.raises(t.IoError, match="cannot open .* for writing"):
        t.save_dataset(ds, str(tmp_path / "no_dir" / "x.json"))


def _random_dataset(t, rng, labeled, ragged):
    d = int(rng.integers(1, 5))
    n = int(rng.integers(1, 20))
    sers = []
    for _ in range(n):
        L = int(rng.integers(1, 30)) if ragged else 7
        x = rng.standard_normal((L, d)) * 10.0 ** rng.integers(-300, 300)
        x[rng.random((L, d)) < 0.05] = -0.0
        x[rng.random((L, d)) < 0.05] = 5e-324
        sers.append(x)
    labels = [f"c{int(rng.integers(0, 5))}-é\"\\\n" for _ in range(n)] if labeled else None
    meta = {"seed": str(int(rng.integers(0, 1 << 30))), "kéy": "v\t€"}
    return t.Dataset(sers if ragged else np.stack(sers), labels, meta)


def test_save_load_round_trip(tsw_host, tmp_path):
    t = tsw_host
    rng = np.random.default_rng(3)
    p = str(tmp_path / "rt.json")
    for it in range(30):
        ds = _random_dataset(t, rng, it % 2 == 0, it % 3 != 0)
        t.save_dataset(ds, p)
        ds2 = t.load_dataset(p)
        a, la = _flat(ds)
        b, lb = _flat(ds2)
        assert la == lb and np.array_equal(a.view(np.uint64), b.view(np.uint64))
        assert ds2.labels == ds.labels and ds2.meta == ds.meta


def test_round_trip_with_live_reference(tsw_host, tmp_path):
    import oracle

    try:
        rio = oracle.ref_io()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference dataset-file library unavailable: {e}")
    t = tsw_host
    rng = np.random.default_rng(4)
    p1, p2 = str(tmp_path / "ours.json"), str(tmp_path / "ref.json")
    for it in range(30):
        ds = _random_dataset(t, rng, it % 2 == 1, it % 3 != 1)
        a, la = _flat(ds)
        t.save_dataset(ds, p1)                   # ours -> reference load
        vals, lens, d, labels, meta = rio.load(p1)
        assert np.array_equal(vals.view(np.uint64), a.view(np.uint64)) and list(lens) == la
        assert labels == ds.labels and meta == ds.meta and d == ds.dim
        rio.resave(p1, p2)                       # reference save -> our load
        ds3 = t.load_dataset(p2)
        b, lb = _flat(ds3)
        assert np.array_equal(b.view(np.uint64), a.view(np.uint64)) and lb == la
        assert ds3.labels == ds.labels and ds3.meta == ds.meta


@pytest.mark.gpu
def test_loaded_file_store_knn(tsw, best_oracle, tmp_path):
    import oracle

    rng = np.random.default_rng(5)
    X = rng.standard_normal((300, 40, 3)).cumsum(1)
    ds = tsw.Dataset(X, [str(i % 4) for i in range(300)], {"src": "test"})
    p = str(tmp_path / "db.json")
    tsw.save_dataset(ds, p)
    ds2 = tsw.load_dataset(p)
    Q = rng.standard_normal((4, 40, 3)).cumsum(1)
    for metric in ("dtw", "dk"):
        gi, gd, _ = tsw.knn(ds2, Q, 3, metric, 4)
        for q in range(len(Q)):
            oi, od, _ = best_oracle.knn(Q[q], oracle.Dataset(X), 3, metric, 4)
            assert np.array_equal(gi[q], oi) and np.array_equal(gd[q], od)
