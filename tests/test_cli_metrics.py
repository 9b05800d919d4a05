"""Experiment drivers and the command line (metrics.hpp:56-72, SPEC.md CLI).

CPU: the CLI's usage contract (exit 2 for usage errors, 1 for runtime errors, messages on
standard error).  GPU: `tswarp_b200 knn` prints the reference's neighbours (rank, index, label,
distance bits), `bench accuracy` equals the leave-one-out accuracy computed from the CPU
oracle's brute force, `bench pruning` lies in [0, 1] and equals the C++ and Python drivers.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1811_11076_b200", "lib", "tswarp_b200")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    import paper_1811_11076_b200 as t

    d = tmp_path_factory.mktemp("cli")
    rng = np.random.default_rng(9)
    protos = rng.standard_normal((3, 30, 2)).cumsum(1)
    X = np.concatenate([protos[c] + 0.3 * rng.standard_normal((20, 30, 2)) for c in range(3)])
    labels = [f"class{c}" for c in range(3) for _ in range(20)]
    data = t.Dataset(X, labels, {"src": "cli-test"})
    q = t.Dataset(np.stack([X[7] + 0.01, protos[1]]))
    t.save_dataset(data, str(d / "data.json"))
    t.save_dataset(q, str(d / "query.json"))
    return str(d / "data.json"), str(d / "query.json"), X, labels


def test_cli_usage_errors(files):
    data, query, _, _ = files
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    r = run("knn", "--metric", "dtw", "--k", "1", "--subsequence", "--query", query, "--data", data)
    assert r.returncode == 2 and "subsequence" in r.stderr
    r = run("knn", "--metric", "manhattan", "--k", "1", "--query", query, "--data", data)
    assert r.returncode == 2
    r = run("knn", "--metric", "dk", "--k", "x", "--query", query, "--data", data)
    assert r.returncode == 2
    r = run("knn", "--metric", "dk", "--k", "1", "--query", query, "--data", data, "--bogus", "1")
    assert r.returncode == 2 and "unknown flag" in r.stderr
    r = run("bench", "lemmas", "--data", data)
    assert r.returncode == 2
    r = run("knn", "--metric", "dk", "--k", "1", "--query", query, "--data", data + ".missing")
    assert r.returncode == 1 and "cannot open" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("metric,sub", [("dtw", False), ("dk", False), ("dk", True)])
def test_cli_knn_matches_reference(files, best_oracle, metric, sub):
    import oracle

    data, query, X, labels = files
    args = ["knn", "--metric", metric, "--k", "4", "--query", query, "--data", data]
    if metric == "dtw":
        args += ["--band", "3"]
    if sub:
        args += ["--subsequence"]
    r = run(*args)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[-1].startswith("counters,")
    oi, od, _ = best_oracle.knn(X[7] + 0.01, oracle.Dataset(X), 4, "dk_sub" if sub else metric, 3)
    for rank, (ln, i, dist) in enumerate(zip(lines[:-1], oi, od), start=1):
        f = ln.split(",")
        assert int(f[0]) == rank and int(f[1]) == int(i) and f[2] == labels[int(i)]
        assert float(f[3]) == dist


@pytest.mark.gpu
def test_bench_accuracy_and_pruning(files, port):
    import oracle
    import paper_1811_11076_b200 as t

    data, query, X, labels = files
    for metric in ("dtw", "dk"):
        r = run("bench", "accuracy", "--data", data, "--metric", metric, "--band", "3")
        assert r.returncode == 0, r.stderr
        acc = float(r.stdout.strip().splitlines()[1].split(",")[1])
        # brute force LOO with the CPU oracle
        correct = 0
        for i in range(len(X)):
            others = [j for j in range(len(X)) if j != i]
            oi, _, _ = port.knn(X[i], oracle.Dataset(X[others]), 1, metric, 3)
            correct += labels[others[int(oi[0])]] == labels[i]
        assert acc == correct / len(X)
        assert t.loo_accuracy(t.load_dataset(data), metric, 3) == acc
    r = run("bench", "pruning", "--data", data, "--query", query, "--band", "3")
    assert r.returncode == 0, r.stderr
    pp = float(r.stdout.strip().splitlines()[1].split(",")[1])
    assert 0.0 <= pp <= 1.0
    assert pp == t.pruning_power(t.load_dataset(query), t.load_dataset(data), 3)
    # the reference's own counters (knn_dtw, k = 1) give the same fraction exactly
    qs = t.load_dataset(query)
    ods = oracle.Dataset(X)
    pruned = sum(int(port.knn(qs.series(i), ods, 1, "dtw", 3)[2][1]) for i in range(len(qs)))
    assert pp == pruned / (len(qs) * len(X))
    r = run("bench", "speedup", "--data", data, "--query", query, "--band", "3", "--reps", "2")
    assert r.returncode == 0 and float(r.stdout.strip().splitlines()[1].split(",")[1]) > 0
