"""CPU: the C-ABI library loads, exports every symbol include/tswarp_b200.h declares, validates
arguments like the reference, and refuses to compute without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1811_11076_b200 as t
from paper_1811_11076_b200 import tswarp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tswarp_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsw_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = t.lib()
    names = declared()
    assert len(names) >= 20
    nm = subprocess.run(["nm", "-D", "--defined-only", tswarp.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tsw_[a-z0-9_]+)\b", nm))
    missing = [n for n in names if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    for n in names:
        assert getattr(lib, n) is not None


def test_python_binding_sets_argtypes_for_every_function_with_arguments():
    lib = t.lib()
    no_args = {"tsw_last_error", "tsw_version", "tsw_device_count"}
    for n in declared():
        if n in no_args:
            continue
        assert getattr(lib, n).argtypes is not None, f"{n}: ctypes argtypes not declared " \
                                                      "(64-bit pointers would be truncated)"


def test_no_cpu_fallback_without_gpu():
    if t.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(t.TswError, match="no CUDA device"):
        t.Store(np.zeros((3, 4, 2)))
    with pytest.raises(t.TswError):
        t.envelope(np.zeros((4, 1)), 1)
    with pytest.raises(t.TswError):
        t.fp64_peak()


def test_store_validation_mirrors_reference():
    # ValidationError before any device work (timeseries.cpp:10-45)
    with pytest.raises(t.ValidationError, match="non-finite"):
        t.Store(np.array([[[0.0], [np.inf]]]))
    with pytest.raises(t.ValidationError, match="at least one series"):
        t.Store([])
    with pytest.raises(t.ValidationError, match="dimensionality"):
        t.Store([np.zeros((3, 2)), np.zeros((3, 1))])
    lib = t.lib()
    out = C.c_void_p()
    v = np.zeros(4)
    assert lib.tsw_store_create(v.ctypes.data_as(C.POINTER(C.c_double)), None, 2, 0, 2, 0,
                                C.byref(out)) == 4  # n == 0 -> TSW_EVALIDATION
    assert b"at least one series" in lib.tsw_last_error()
    assert lib.tsw_store_create(v.ctypes.data_as(C.POINTER(C.c_double)), None, 2, 2, 0, 0,
                                C.byref(out)) == 4  # d == 0
    assert lib.tsw_knn(None, None, 1, 1, 0, 0, 1, None, None) == 1  # null store -> TSW_EINVAL


def test_query_validation_mirrors_reference():
    ds = t.Dataset(np.zeros((4, 6, 2)))
    with pytest.raises(ValueError, match="k must be positive"):
        t.knn_dtw(np.zeros((6, 2)), ds, 0, 1)
    with pytest.raises(ValueError, match="query dim 3 != dataset dim 2"):
        t.knn_dk(np.zeros((6, 3)), ds, 1)
    with pytest.raises(ValueError, match="length differs from the query"):
        t.knn_dtw(np.zeros((5, 2)), ds, 1, 1)
    with pytest.raises(ValueError, match="eps must be nonnegative"):
        t.epsnn_dk(np.zeros((6, 2)), ds, -0.5)


def test_synth_configs_shapes_and_determinism():
    for cfg, (n, L, d, r, k, q) in {1: (2000, 128, 2, 13, 1, 16), 2: (20000, 128, 3, 13, 1, 64),
                                    3: (50000, 256, 2, 26, 5, 256), 4: (100000, 256, 16, 26, 1, 32),
                                    5: (200000, 1024, 3, 51, 10, 32)}.items():
        sh0, sh1 = t.synth_shape(cfg, 0), t.synth_shape(cfg, 1)
        assert (sh0["count"], sh0["len"], sh0["d"], sh0["r"], sh0["k"]) == (n, L, d, r, k)
        assert sh1["count"] == q
    a, la = t.synth(3, 1, seed=7)
    b, lb = t.synth(3, 1, seed=7)
    c, _ = t.synth(3, 1, seed=8)
    assert np.array_equal(a, b) and np.array_equal(la, lb) and not np.array_equal(a, c)
    assert sorted(set(la.tolist())) == list(range(20))
    # per-series, per-dimension z-normalisation (population SD)
    np.testing.assert_allclose(a.mean(axis=1), 0.0, atol=1e-12)
    np.testing.assert_allclose(a.std(axis=1), 1.0, atol=1e-12)
    q2, _ = t.synth(2, 1)
    assert q2.shape == (64, 128, 3)
    np.testing.assert_allclose(q2.std(axis=1), 1.0, atol=1e-12)


def test_cpp_dropin_header_compiles_and_links(tmp_path):
    """The C++ drop-in API (include/tswarp_b200.hpp) builds a reference-style caller."""
    src = tmp_path / "caller.cpp"
    src.write_text(DROPIN_CALLER)
    exe = tmp_path / "caller"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe), "-L", os.path.dirname(tswarp.LIB_PATH), "-ltswarp_b200",
                    f"-Wl,-rpath,{os.path.dirname(tswarp.LIB_PATH)}"], check=True)
    assert exe.exists()


DROPIN_CALLER = r"""
#include <cstdio>
#include <vector>
#include "tswarp_b200.hpp"
int main() {
    using namespace tswarp;
    std::vector<TimeSeries> s;
    for (int i = 0; i < 8; ++i) s.emplace_back(std::vector<double>{0.0 + i, 1.0, 2.0 * i, 3.0}, 2);
    Dataset data(std::move(s));
    TimeSeries q(std::vector<double>{1.0, 1.0, 2.0, 3.0}, 2);
    try {
        SearchReport a = knn_dtw(q, data, 3, BandRadius{1});
        SearchReport b = knn_dk(q, data, 3);
        for (const auto& nb : a.neighbors) std::printf("dtw %zu %.17g\n", nb.index, nb.distance);
        for (const auto& nb : b.neighbors) std::printf("dk %zu %.17g\n", nb.index, nb.distance);
        std::printf("counters %zu %zu %zu %zu\n", a.counters.lb_computed, a.counters.lb_pruned,
                    a.counters.full_dp, a.counters.early_abandoned);
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 3;
    }
    return 0;
}
"""
