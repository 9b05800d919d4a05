"""Python mirror of the reference query API over the tswarp_b200 C ABI (ctypes).

Same names, argument meaning and error behaviour as the reference's hot-path API
(proj/core/include/tswarp/search.hpp:13-63, types.hpp:14-121):

* ``knn_dtw(query, data, k, r, threads=1)``   <-> ``tswarp::knn_dtw``   (search.cpp:125-169)
* ``knn_dk(query, data, k, threads=1)``       <-> ``tswarp::knn_dk``    (search.cpp:171-214)
* ``epsnn_dk(query, data, eps, threads=1)``   <-> ``tswarp::epsnn_dk``  (search.cpp:216-239)
* ``knn_dk_sub(query, data, k, threads=1)``   <-> ``tswarp::knn_dk_sub`` (search.cpp:250-280)
* ``sub_search_dk(query, haystack, eps)``     <-> ``tswarp::sub_search_dk`` (search.cpp:241-248)
* ``sparse_dk_sub(s, t, eps)``                <-> ``tswarp::sparse_dk_sub`` (dogkeeper.cpp:235-241)
* ``SearchReport`` / ``SearchCounters`` / ``Neighbor`` mirror search.hpp:13-32.
* ``ValidationError`` mirrors tswarp::ValidationError; invalid arguments raise ``ValueError``
  (the Python spelling of std::invalid_argument).

Series are numpy arrays of shape [length, dim] (row-major, exactly TimeSeries::flat()).
A ``Dataset`` uploads its series once into a device store on first use.

There is no CPU fallback: importing works anywhere, but every compute call raises
``RuntimeError`` unless libtswarp_b200.so is built and a CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# TSW_LIB: an alternative build of the same library (A/B measurements of compile-time variants)
LIB_PATH = os.environ.get("TSW_LIB") or os.path.join(HERE, "lib", "libtswarp_b200.so")

METRIC_DTW = 0
METRIC_DK = 1
METRIC_DK_SUB = 2
_METRICS = {"dtw": METRIC_DTW, "dk": METRIC_DK, "dk_sub": METRIC_DK_SUB}


def _metric(name: str) -> int:
    try:
        return _METRICS[name]
    except KeyError:
        raise ValueError(f"unknown metric {name!r} (dtw | dk | dk_sub)") from None

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_uint64)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


class ValidationError(ValueError):
    """tswarp::ValidationError (types.hpp:25-28)."""


class TswError(RuntimeError):
    pass


class ParseError(RuntimeError):
    """tswarp::ParseError (types.hpp:19-22): malformed dataset files."""


class IoError(RuntimeError):
    """tswarp::IoError (types.hpp:31-34): dataset files that cannot be read or written."""


class Neighbor_t(C.Structure):
    _fields_ = [("index", C.c_uint64), ("distance", C.c_double)]


class Counters_t(C.Structure):
    _fields_ = [("lb_computed", C.c_uint64), ("lb_pruned", C.c_uint64), ("full_dp", C.c_uint64),
                ("early_abandoned", C.c_uint64), ("gdk_calls", C.c_uint64)]


class Stats_t(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_envelope", C.c_double), ("ms_bound", C.c_double),
                ("ms_select", C.c_double), ("ms_probe_dp", C.c_double),
                ("ms_compact", C.c_double), ("ms_dp", C.c_double),
                ("bound_bytes", C.c_uint64), ("bound_passes", C.c_uint64),
                ("dp_pairs", C.c_uint64), ("dp_cells", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("bound_block", C.c_uint64)]


_lib = None


def lib():
    """Load libtswarp_b200.so (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TswError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                       " or `make -C paper_1811_11076_b200/csrc`")
    L = C.CDLL(LIB_PATH)
    L.tsw_last_error.restype = C.c_char_p
    L.tsw_version.restype = C.c_int
    L.tsw_device_count.restype = C.c_int
    L.tsw_store_create.argtypes = [_dp, _up, _u64, _u64, _u64, C.c_int, C.POINTER(_vp)]
    L.tsw_store_destroy.argtypes = [_vp]
    L.tsw_store_destroy.restype = None
    L.tsw_store_info.argtypes = [_vp, _up, _up, _up, _up, _up]
    L.tsw_knn.argtypes = [_vp, _dp, _u64, _u64, C.c_int, _u64, _u64, C.POINTER(Neighbor_t),
                          C.POINTER(Counters_t)]
    L.tsw_epsnn_dk.argtypes = [_vp, _dp, _u64, C.c_double, C.POINTER(Neighbor_t), _u64, _up,
                               C.POINTER(Counters_t)]
    L.tsw_plan_create.argtypes = [_vp, _u64, _u64, C.c_int, _u64, _u64, C.POINTER(_vp)]
    L.tsw_plan_destroy.argtypes = [_vp]
    L.tsw_plan_destroy.restype = None
    L.tsw_plan_set_queries.argtypes = [_vp, _dp, _u64, _vp]
    L.tsw_plan_set_queries_device.argtypes = [_vp, _vp, _u64, _vp]
    L.tsw_plan_execute.argtypes = [_vp, _vp]
    L.tsw_plan_fetch.argtypes = [_vp, C.POINTER(Neighbor_t), C.POINTER(Counters_t), _vp]
    L.tsw_plan_set_timing.argtypes = [_vp, C.c_int]
    L.tsw_plan_set_graph.argtypes = [_vp, C.c_int]
    L.tsw_plan_stats.argtypes = [_vp, C.POINTER(Stats_t)]
    L.tsw_envelope.argtypes = [_dp, _u64, _u64, _u64, _dp, _dp]
    L.tsw_lb_box_all.argtypes = [_vp, _dp, _u64, _u64, _dp, _dp]
    L.tsw_dist_all.argtypes = [_vp, _dp, _u64, C.c_int, _u64, C.c_double, _ip, _dp]
    L.tsw_lb_box_exact_all.argtypes = [_vp, _dp, _u64, _u64, _dp]
    L.tsw_pruning_power.argtypes = [_vp, _dp, _u64, _u64, _u64, C.POINTER(C.c_double), _up]
    L.tsw_sub_dk_all.argtypes = [_vp, _dp, _u64, C.c_double, _ip, _dp, _up]
    L.tsw_last_transfer_bytes.argtypes = [_up, _up]
    L.tsw_fp64_peak.argtypes = [_dp]
    L.tsw_l2_flush.argtypes = [_vp, _u64, _vp]
    L.tsw_dataset_load_json.argtypes = [C.c_char_p, C.POINTER(_vp)]
    L.tsw_dataset_free.argtypes = [_vp]
    L.tsw_dataset_free.restype = None
    L.tsw_dataset_info.argtypes = [_vp, _up, _up, _up, _ip, _up]
    L.tsw_dataset_values.argtypes = [_vp]
    L.tsw_dataset_values.restype = _dp
    L.tsw_dataset_lengths.argtypes = [_vp]
    L.tsw_dataset_lengths.restype = _up
    L.tsw_dataset_label.argtypes = [_vp, _u64]
    L.tsw_dataset_label.restype = C.c_char_p
    L.tsw_dataset_meta.argtypes = [_vp, _u64, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]
    L.tsw_dataset_to_store.argtypes = [_vp, C.c_int, C.POINTER(_vp)]
    L.tsw_dataset_save_json.argtypes = [C.c_char_p, _dp, _up, _u64, _u64, C.POINTER(C.c_char_p),
                                        C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), _u64]
    L.tsw_synth_shape.argtypes = [C.c_int, C.c_int, _up, _up, _up, _up, _up]
    L.tsw_synth_generate.argtypes = [C.c_int, C.c_int, _u64, _dp, C.POINTER(C.c_int32)]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().tsw_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 4:
        raise ValidationError(msg)
    if rc == 2:
        raise MemoryError(msg)
    if rc == 5:
        raise ParseError(msg)
    if rc == 6:
        raise IoError(msg)
    raise TswError(msg)


def device_count() -> int:
    return int(lib().tsw_device_count())


def last_transfer_bytes() -> tuple[int, int]:
    h2d, d2h = _u64(), _u64()
    lib().tsw_last_transfer_bytes(C.byref(h2d), C.byref(d2h))
    return h2d.value, d2h.value


def fp64_peak() -> float:
    """Measured FP64 DADD/DMUL throughput of the current device, lane-ops per second."""
    v = C.c_double()
    _check(lib().tsw_fp64_peak(C.byref(v)))
    return v.value


def l2_flush(dev_ptr: int, nbytes: int, stream: int | None = None) -> None:
    _check(lib().tsw_l2_flush(dev_ptr, nbytes, stream))


def _series(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.ndim != 2:
        raise ValueError("a series is a [length, dim] array")
    return a


# ---- result types (search.hpp:13-32) ---------------------------------------------------------
@dataclass
class SearchCounters:
    lb_computed: int = 0
    lb_pruned: int = 0
    full_dp: int = 0
    early_abandoned: int = 0
    gdk_calls: int = 0


@dataclass
class Neighbor:
    index: int
    distance: float


@dataclass
class SearchReport:
    neighbors: list = field(default_factory=list)
    counters: SearchCounters = field(default_factory=SearchCounters)
    wall_time_seconds: float = 0.0


# ---- the device store -------------------------------------------------------------------
class Store:
    """A device-resident, read-only candidate store (tsw_store)."""

    def __init__(self, series, device: int = 0):
        L = lib()
        if isinstance(series, np.ndarray) and series.ndim == 3:
            vals = np.ascontiguousarray(series, dtype=np.float64)
            n, ln, d = vals.shape
            lengths = None
            uniform = ln
        else:
            arrs = [_series(s) for s in series]
            if not arrs:
                raise ValidationError("dataset must contain at least one series")
            d = arrs[0].shape[1]
            for i, a in enumerate(arrs):
                if a.shape[1] != d:
                    raise ValidationError(f"series {i} has dimensionality {a.shape[1]}, dataset has {d}")
            n = len(arrs)
            vals = np.concatenate([a.reshape(-1) for a in arrs]) if n else np.zeros(0)
            lengths = np.array([a.shape[0] for a in arrs], dtype=np.uint64)
            uniform = 0
        self.n, self.dim = int(n), int(d)
        self.lengths = lengths
        h = _vp()
        _check(L.tsw_store_create(vals.ctypes.data_as(_dp),
                                  lengths.ctypes.data_as(_up) if lengths is not None else None,
                                  uniform, n, d, device, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def info(self):
        n, d, ml, ul, by = (_u64(), _u64(), _u64(), _u64(), _u64())
        _check(lib().tsw_store_info(self._h, C.byref(n), C.byref(d), C.byref(ml), C.byref(ul),
                                    C.byref(by)))
        return dict(n=n.value, d=d.value, max_len=ml.value, uniform_len=ul.value,
                    device_bytes=by.value)

    def close(self):
        if getattr(self, "_h", None):
            lib().tsw_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Dataset:
    """Mirror of tswarp::Dataset: validated series plus a lazily uploaded device store."""

    def __init__(self, series, labels: Sequence[str] | None = None, meta: dict | None = None):
        if isinstance(series, np.ndarray) and series.ndim == 3:
            self._arr = np.ascontiguousarray(series, dtype=np.float64)
            self._list = None
            self.n, _, self.dim = self._arr.shape
        else:
            self._list = [_series(s) for s in series]
            self._arr = None
            if not self._list:
                raise ValidationError("dataset must contain at least one series")
            self.n, self.dim = len(self._list), self._list[0].shape[1]
        if self.n == 0:
            raise ValidationError("dataset must contain at least one series")
        self.labels = list(labels) if labels is not None else None
        self.meta = dict(meta) if meta else {}
        self._store: Store | None = None

    def __len__(self):
        return self.n

    def length(self, i: int) -> int:
        return self._arr.shape[1] if self._arr is not None else self._list[i].shape[0]

    @property
    def store(self) -> Store:
        if self._store is None:
            self._store = Store(self._arr if self._arr is not None else self._list)
        return self._store


def series(self, i: int) -> np.ndarray:
    return self._arr[i] if self._arr is not None else self._list[i]


Dataset.series = series


# ---- dataset files (dataset_io.hpp:9-23) ---------------------------------------------------
def load_dataset(path) -> Dataset:
    """tswarp::load_dataset(path) -- dataset_io.cpp:45-112: ParseError / ValidationError /
    IoError as the reference raises them."""
    L = lib()
    h = _vp()
    _check(L.tsw_dataset_load_json(os.fsencode(path), C.byref(h)))
    try:
        n, d, tot, nm = _u64(), _u64(), _u64(), _u64()
        lab = C.c_int()
        _check(L.tsw_dataset_info(h, C.byref(n), C.byref(d), C.byref(tot), C.byref(lab), C.byref(nm)))
        vals = np.ctypeslib.as_array(L.tsw_dataset_values(h), shape=(tot.value * d.value,)).copy()
        lens = np.ctypeslib.as_array(L.tsw_dataset_lengths(h), shape=(n.value,)).copy()
        labels = [L.tsw_dataset_label(h, i).decode("utf-8") for i in range(n.value)] if lab.value else None
        meta = {}
        for i in range(nm.value):
            k, v = C.c_char_p(), C.c_char_p()
            _check(L.tsw_dataset_meta(h, i, C.byref(k), C.byref(v)))
            meta[k.value.decode("utf-8")] = v.value.decode("utf-8")
    finally:
        L.tsw_dataset_free(h)
    offs = np.concatenate([[0], np.cumsum(lens * d.value)]).astype(np.int64)
    sers = [vals[offs[i]:offs[i + 1]].reshape(-1, d.value) for i in range(n.value)]
    if len(set(lens.tolist())) == 1:
        return Dataset(np.stack(sers), labels, meta)
    return Dataset(sers, labels, meta)


def save_dataset(ds: Dataset, path) -> None:
    """tswarp::save_dataset(ds, path) -- dataset_io.cpp:114-140 (round-trip exact numbers)."""
    sers = [np.ascontiguousarray(ds.series(i), dtype=np.float64) for i in range(ds.n)]
    vals = np.concatenate([x.reshape(-1) for x in sers])
    lens = np.array([x.shape[0] for x in sers], dtype=np.uint64)
    labels = None
    if ds.labels is not None:
        labels = (C.c_char_p * ds.n)(*[str(x).encode("utf-8") for x in ds.labels])
    keys = sorted(ds.meta)
    kk = (C.c_char_p * max(1, len(keys)))(*[k.encode("utf-8") for k in keys])
    vv = (C.c_char_p * max(1, len(keys)))(*[str(ds.meta[k]).encode("utf-8") for k in keys])
    _check(lib().tsw_dataset_save_json(os.fsencode(path), vals.ctypes.data_as(_dp),
                                       lens.ctypes.data_as(_up), ds.n, ds.dim, labels, kk, vv,
                                       len(keys)))


# ---- experiment drivers (metrics.hpp:56-72) ---------------------------------------------
def _by_length(data: Dataset):
    groups: dict[int, list[int]] = {}
    for i in range(data.n):
        groups.setdefault(data.length(i), []).append(i)
    return groups


def pruning_power(queries: Dataset, data, r: int) -> float:
    """pruning_power (metrics.hpp:54-56): the fraction of candidate DTW computations the lb_box
    test skips over 1-NN knn_dtw scans of every query, with the reference's own scan schedule
    (64-candidate blocks, block-frozen threshold, search.cpp:139-162) replayed exactly on the
    GPU (tsw_pruning_power) -- deterministic and equal to the reference's counters."""
    st = _as_store(data)
    pruned = total = 0
    for L, ids in _by_length(queries).items():
        qs = np.ascontiguousarray(np.stack([queries.series(i) for i in ids]), dtype=np.float64)
        if qs.shape[2] != st.dim:
            raise ValueError(f"knn_dtw: query dim {qs.shape[2]} != dataset dim {st.dim}")
        per = np.zeros(len(ids), dtype=np.uint64)
        p = C.c_double()
        _check(lib().tsw_pruning_power(st.handle, qs.ctypes.data_as(_dp), len(ids), L, r,
                                       C.byref(p), per.ctypes.data_as(_up)))
        pruned += int(per.sum())
        total += len(ids) * st.n
    return pruned / total if total else 0.0


def lb_box_exact_all(data, query, r: int) -> np.ndarray:
    """The reference's fp64 lb_box(data[i], envelope(query, r)) for every candidate, bit for
    bit (lower_bounds.cpp:19-46) -- not the pipeline's fp32 bound."""
    q = _series(query)
    st = _as_store(data)
    out = np.empty(st.n)
    _check(lib().tsw_lb_box_exact_all(st.handle, q.ctypes.data_as(_dp), q.shape[0], r,
                                      out.ctypes.data_as(_dp)))
    return out


def loo_accuracy(data: Dataset, metric: str = "dtw", r: int = 0) -> float:
    """Leave-one-out 1-NN accuracy (ties to the lowest index); labels required."""
    if data.labels is None:
        raise ValueError("loo_accuracy: the dataset has no labels")
    if data.n < 2:
        raise ValueError("loo_accuracy: needs at least two series")
    correct = 0
    for L, ids in _by_length(data).items():
        qs = np.stack([data.series(i) for i in ids])
        idx, _, _ = knn(data, qs, 2, metric, r)
        for row, i in enumerate(ids):
            j = next(int(x) for x in idx[row] if int(x) != i)
            correct += data.labels[j] == data.labels[i]
    return correct / data.n


def speedup(queries: Dataset, data, r: int, repetitions: int = 3) -> float:
    """Median wall time of the DTW + LB_Box 1-NN scan over that of the dog-keeper scan."""
    def timed(metric):
        def run():
            for L, ids in _by_length(queries).items():
                knn(data, np.stack([queries.series(i) for i in ids]), 1, metric, r)
        run()
        ts = []
        for _ in range(repetitions):
            t0 = time.perf_counter()
            run()
            ts.append(time.perf_counter() - t0)
        return sorted(ts)[len(ts) // 2]
    t_dtw, t_dk = timed("dtw"), timed("dk")
    return t_dtw / t_dk if t_dk > 0 else 0.0


def _as_store(data) -> Store:
    return data.store if isinstance(data, Dataset) else data


# ---- batched k-NN -----------------------------------------------------------------------
def knn(data, queries, k: int, metric: str = "dtw", r: int = 0):
    """Batched k-NN: queries [nq, L, d] -> (indices u64[nq, kk], distances f64[nq, kk],
    counters u64[nq, 5]) with kk = min(k, n).  A query with fewer neighbours (the reference's
    KBest can end short, see TSW_NO_NEIGHBOR) has its row padded with (NO_NEIGHBOR, +inf)."""
    qs = np.ascontiguousarray(queries, dtype=np.float64)
    if qs.ndim == 2:
        qs = qs[None]
    nq, qlen, d = qs.shape
    # argument checks first, as the reference does before touching the data (search.cpp:127)
    if k == 0:
        raise ValueError(f"knn_{metric}: k must be positive")
    if d != data.dim:
        raise ValueError(f"knn_{metric}: query dim {d} != dataset dim {data.dim}")
    st = _as_store(data)
    kk = min(k, st.n)
    out = (Neighbor_t * max(1, nq * kk))()
    ctr = (Counters_t * max(1, nq))()
    m = _metric(metric)
    _check(lib().tsw_knn(st.handle, qs.ctypes.data_as(_dp), nq, qlen, m, r, k, out, ctr))
    raw = np.frombuffer(out, dtype=np.dtype([("index", "<u8"), ("distance", "<f8")]),
                        count=nq * kk)
    idx = raw["index"].reshape(nq, kk).copy()
    dist = raw["distance"].reshape(nq, kk).copy()
    c = np.frombuffer(ctr, dtype=np.uint64, count=nq * 5).reshape(nq, 5).copy()
    return idx, dist, c


NO_NEIGHBOR = np.iinfo(np.uint64).max  # TSW_NO_NEIGHBOR: unused tail entry of a short row


def _report(idx, dist, c, wall) -> SearchReport:
    return SearchReport([Neighbor(int(i), float(v)) for i, v in zip(idx, dist) if i != NO_NEIGHBOR],
                        SearchCounters(*[int(x) for x in c]), wall)


def knn_dtw(query, data, k: int, r, threads: int = 1) -> SearchReport:
    """tswarp::knn_dtw(query, data, k, BandRadius r, threads) -- search.hpp:46-47."""
    rv = r.value if hasattr(r, "value") else int(r)
    q = _series(query)
    if k == 0:
        raise ValueError("knn_dtw: k must be positive")
    _check_query(q, data, True, "knn_dtw")
    t0 = time.perf_counter()
    idx, dist, c = knn(data, q[None], k, "dtw", rv)
    return _report(idx[0], dist[0], c[0], time.perf_counter() - t0)


def knn_dk(query, data, k: int, threads: int = 1) -> SearchReport:
    """tswarp::knn_dk(query, data, k, threads) -- search.hpp:56-57."""
    q = _series(query)
    if k == 0:
        raise ValueError("knn_dk: k must be positive")
    _check_query(q, data, False, "knn_dk")
    t0 = time.perf_counter()
    idx, dist, c = knn(data, q[None], k, "dk")
    return _report(idx[0], dist[0], c[0], time.perf_counter() - t0)


def knn_dk_sub(query, data, k: int, threads: int = 1) -> SearchReport:
    """tswarp::knn_dk_sub(query, data, k, threads) -- search.hpp:75-76: the k candidates whose
    best subsequence match of the query is closest, ranked by (match distance, index)."""
    q = _series(query)
    if k == 0:
        raise ValueError("knn_dk_sub: k must be positive")
    _check_query(q, data, False, "knn_dk_sub")
    t0 = time.perf_counter()
    idx, dist, c = knn(data, q[None], k, "dk_sub")
    return _report(idx[0], dist[0], c[0], time.perf_counter() - t0)


@dataclass
class SubMatch:
    """tswarp::SubMatch (dogkeeper.hpp:11-14)."""
    distance: float
    end_index: int


def sub_dk_all(data, query, eps: float = float("inf")):
    """-> (found bool[n], distance f64[n], end u64[n]): sparse_dk_sub(query, data[i], eps) for
    every candidate (== sub_search_dk, whose greedy seed only tightens eps).  Not found:
    distance = +inf (std::nullopt)."""
    st = _as_store(data)
    q = _series(query)
    if q.shape[1] != st.dim:
        raise ValueError("sub_search_dk: dimensionality mismatch")
    if eps < 0:
        raise ValueError("sparse_dk_sub: eps must be nonnegative")
    found = np.empty(st.n, dtype=np.int32)
    val = np.empty(st.n)
    end = np.empty(st.n, dtype=np.uint64)
    _check(lib().tsw_sub_dk_all(st.handle, q.ctypes.data_as(_dp), q.shape[0], float(eps),
                                found.ctypes.data_as(_ip), val.ctypes.data_as(_dp),
                                end.ctypes.data_as(_up)))
    return found.astype(bool), val, end


def sparse_dk_sub(s, t, eps: float):
    """tswarp::sparse_dk_sub(s, t, eps) -- dogkeeper.hpp:72-73: SubMatch or None (nullopt)."""
    s, t = _series(s), _series(t)
    if s.shape[1] != t.shape[1]:
        raise ValueError(f"sparse_dk_sub: dimensionality mismatch ({s.shape[1]} vs {t.shape[1]})")
    if eps < 0:
        raise ValueError("sparse_dk_sub: eps must be nonnegative")
    f, v, e = sub_dk_all(Store([t]), s, eps)
    return SubMatch(float(v[0]), int(e[0])) if f[0] else None


def sub_search_dk(query, haystack, eps: float = float("inf")):
    """tswarp::sub_search_dk(query, haystack, eps) -- search.hpp:68-69."""
    q, h = _series(query), _series(haystack)
    if q.shape[1] != h.shape[1]:
        raise ValueError("sub_search_dk: dimensionality mismatch")
    return sparse_dk_sub(q, h, eps)


def epsnn_dk(query, data, eps: float, threads: int = 1) -> SearchReport:
    """tswarp::epsnn_dk(query, data, eps, threads) -- search.hpp:61-62."""
    q = _series(query)
    if eps < 0:
        raise ValueError("epsnn_dk: eps must be nonnegative")
    _check_query(q, data, False, "epsnn_dk")
    st = _as_store(data)
    out = (Neighbor_t * st.n)()
    cnt = _u64()
    ctr = Counters_t()
    t0 = time.perf_counter()
    _check(lib().tsw_epsnn_dk(st.handle, q.ctypes.data_as(_dp), q.shape[0], float(eps), out,
                              st.n, C.byref(cnt), C.byref(ctr)))
    n = cnt.value
    nb = [Neighbor(int(out[j].index), float(out[j].distance)) for j in range(n)]
    return SearchReport(nb, SearchCounters(ctr.lb_computed, ctr.lb_pruned, ctr.full_dp,
                                           ctr.early_abandoned, ctr.gdk_calls),
                        time.perf_counter() - t0)


def _check_query(q, data, equal_lengths, op):
    """check_query, search.cpp:99-115."""
    n = data.n
    dim = data.dim
    if q.shape[1] != dim:
        raise ValueError(f"{op}: query dim {q.shape[1]} != dataset dim {dim}")
    if equal_lengths and isinstance(data, Dataset):
        if data._arr is not None:  # uniform-length dataset: one comparison
            if n and data._arr.shape[1] != q.shape[0]:
                raise ValueError(f"{op}: series 0 length differs from the query (lower bounds "
                                 "require equal lengths)")
            return
        for i in range(n):
            if data.length(i) != q.shape[0]:
                raise ValueError(f"{op}: series {i} length differs from the query (lower bounds "
                                 "require equal lengths)")


# ---- single operators (parity / diagnostics) --------------------------------------------
def envelope(series, r: int):
    s = _series(series)
    lo = np.empty_like(s)
    hi = np.empty_like(s)
    _check(lib().tsw_envelope(s.ctypes.data_as(_dp), s.shape[0], s.shape[1], r,
                              lo.ctypes.data_as(_dp), hi.ctypes.data_as(_dp)))
    return lo, hi


def lb_box_all(data, query, r: int):
    """-> (lb, ub): the fp32 directed-rounded LB_Box lower bound of every candidate (K2; a
    rigorous lower bound of lb_box(data[i], envelope(query, r))) and the diagonal DTW upper
    bound used to seed the threshold."""
    st = _as_store(data)
    q = _series(query)
    lb = np.empty(st.n)
    ub = np.empty(st.n)
    _check(lib().tsw_lb_box_all(st.handle, q.ctypes.data_as(_dp), q.shape[0], r,
                                lb.ctypes.data_as(_dp), ub.ctypes.data_as(_dp)))
    return lb, ub


def dist_all(data, query, metric: str, r: int = 0, eps: float = float("inf")):
    """-> (exact bool[n], value f64[n]) : dtw_early_abandon / sparse_dk for every candidate."""
    st = _as_store(data)
    q = _series(query)
    ex = np.empty(st.n, dtype=np.int32)
    val = np.empty(st.n)
    _check(lib().tsw_dist_all(st.handle, q.ctypes.data_as(_dp), q.shape[0],
                              METRIC_DTW if metric == "dtw" else METRIC_DK, r, float(eps),
                              ex.ctypes.data_as(_ip), val.ctypes.data_as(_dp)))
    return ex.astype(bool), val


# ---- plans (device-resident batched execution) ------------------------------------------
class Plan:
    def __init__(self, data, nq_max: int, qlen: int, metric: str, r: int, k: int):
        self.store = _as_store(data)
        self.metric = metric
        self.k = k
        self.kk = min(k, self.store.n)
        h = _vp()
        _check(lib().tsw_plan_create(self.store.handle, nq_max, qlen, _metric(metric), r, k,
                                     C.byref(h)))
        self._h = h
        self.nq = 0
        self._qkeep = None

    def set_queries(self, queries: np.ndarray, stream: int | None = None):
        qs = np.ascontiguousarray(queries, dtype=np.float64)
        self._qkeep = qs  # keep alive during async copy
        self.nq = qs.shape[0]
        _check(lib().tsw_plan_set_queries(self._h, qs.ctypes.data_as(_dp), self.nq, stream))

    def set_queries_device(self, ptr: int, nq: int, stream: int | None = None):
        self.nq = nq
        _check(lib().tsw_plan_set_queries_device(self._h, ptr, nq, stream))

    def execute(self, stream: int | None = None):
        _check(lib().tsw_plan_execute(self._h, stream))

    def fetch(self, stream: int | None = None):
        out = (Neighbor_t * max(1, self.nq * self.kk))()
        ctr = (Counters_t * max(1, self.nq))()
        _check(lib().tsw_plan_fetch(self._h, out, ctr, stream))
        raw = np.frombuffer(out, dtype=np.dtype([("index", "<u8"), ("distance", "<f8")]),
                            count=self.nq * self.kk)
        c = np.frombuffer(ctr, dtype=np.uint64, count=self.nq * 5).reshape(self.nq, 5).copy()
        return (raw["index"].reshape(self.nq, self.kk).copy(),
                raw["distance"].reshape(self.nq, self.kk).copy(), c)

    def set_graph(self, on: bool):
        """Run executions as one captured CUDA graph (re-captured on shape/stream change)."""
        _check(lib().tsw_plan_set_graph(self._h, 1 if on else 0))

    def set_timing(self, on: bool):
        _check(lib().tsw_plan_set_timing(self._h, 1 if on else 0))

    def stats(self) -> dict:
        s = Stats_t()
        _check(lib().tsw_plan_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats_t._fields_}

    def close(self):
        if getattr(self, "_h", None):
            lib().tsw_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- seeded synthetic inputs (BASELINE.json configs 1..5) --------------------------------
def synth_shape(config: int, part: int = 0) -> dict:
    vals = [_u64() for _ in range(5)]
    _check(lib().tsw_synth_shape(config, part, *[C.byref(v) for v in vals]))
    return dict(zip(["count", "len", "d", "r", "k"], [v.value for v in vals]))


def synth(config: int, part: int, seed: int = 20181127):
    """-> (values f64[count, len, d], labels i32[count])"""
    sh = synth_shape(config, part)
    out = np.empty((sh["count"], sh["len"], sh["d"]), dtype=np.float64)
    lab = np.empty(sh["count"], dtype=np.int32)
    _check(lib().tsw_synth_generate(config, part, seed, out.ctypes.data_as(_dp),
                                    lab.ctypes.data_as(C.POINTER(C.c_int32))))
    return out, lab
