"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU oracles of the hot path.

* ``port()`` -- oracle/tswarp_oracle.c, the plain-C restatement (always buildable: gcc).
* ``ref()``  -- the reference's own sources compiled by oracle/Makefile into
  oracle/_ref/libtswarp_ref.so (needs /root/reference at build time; the built .so travels to
  the GPU box with the repo snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference / cpu_baseline legs may
import this package, and only as the checker or the CPU baseline -- never as the product.
Both expose the same Python surface (class ``Oracle``), so every parity test can run against
either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libtswarp_ref.so")
REF_IO_SO = os.path.join(HERE, "_ref", "libtswarp_ref_io.so")
SYNTH_SO = os.path.join(HERE, "_build", "libtsw_synth.so")
REF_ROOT = "/root/reference/proj/core"

_METRIC = {"dtw": 0, "dk": 1, "dk_sub": 2}

_lock = threading.Lock()
_cache: dict[str, "Oracle"] = {}

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_uint64)
_ip = C.POINTER(C.c_int)


def build(ref: bool | None = None) -> None:
    """Build the port (always) and the reference library (when /root/reference exists)."""
    targets = ["port"]
    if ref or (ref is None and os.path.isdir(REF_ROOT)):
        targets += ["ref", "ref_io"]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _uptr(a: np.ndarray):
    return a.ctypes.data_as(_up)


class OracleError(RuntimeError):
    pass


class Dataset:
    """Concatenated row-major values + per-series lengths (points), as the oracles take them."""

    def __init__(self, series: Sequence[np.ndarray] | np.ndarray):
        if isinstance(series, np.ndarray) and series.ndim == 3:
            n, L, d = series.shape
            self.values = np.ascontiguousarray(series, dtype=np.float64).reshape(-1)
            self.lengths = np.full(n, L, dtype=np.uint64)
            self.dim = d
        else:
            arrs = [np.ascontiguousarray(s, dtype=np.float64) for s in series]
            self.dim = arrs[0].shape[1]
            self.values = np.concatenate([a.reshape(-1) for a in arrs])
            self.lengths = np.array([a.shape[0] for a in arrs], dtype=np.uint64)
        self.n = len(self.lengths)
        self._ref_handle = None
        self._ref_lib = None

    def ref_handle(self, lib):
        if self._ref_handle is None:
            h = lib.ref_dataset_create(_dptr(self.values), _uptr(self.lengths), self.n, self.dim)
            if not h:
                raise OracleError(lib.ref_last_error().decode())
            self._ref_handle, self._ref_lib = h, lib
        return self._ref_handle

    def __del__(self):
        if self._ref_handle is not None:
            try:
                self._ref_lib.ref_dataset_destroy(self._ref_handle)
            except Exception:
                pass


class Oracle:
    def __init__(self, path: str, kind: str):
        self.kind = kind  # "port" | "reference"
        self.lib = C.CDLL(path)
        p = "orc_" if kind == "port" else "ref_"
        self.p = p
        L = self.lib
        if kind == "reference":
            L.ref_last_error.restype = C.c_char_p
            L.ref_dataset_create.restype = C.c_void_p
            L.ref_dataset_create.argtypes = [_dp, _up, _u64, _u64]
            L.ref_dataset_destroy.argtypes = [C.c_void_p]
            L.ref_knn.argtypes = [C.c_void_p, _dp, _u64, _u64, C.c_int, _u64, _u64, C.c_int, _u64,
                                  _up, _dp, _up, _up, _dp]
            L.ref_knn_batch.argtypes = [C.c_void_p, _dp, _u64, _u64, _u64, C.c_int, _u64, _u64,
                                        C.c_int, _u64, _up, _dp, _up, _up]
            L.ref_epsnn_dk.argtypes = [C.c_void_p, _dp, _u64, _u64, C.c_double, C.c_int, _u64,
                                       _up, _dp, _up, _up]
        else:
            L.orc_knn_dtw.argtypes = [_dp, _u64, _u64, _dp, _up, _u64, _u64, _u64, _u64, _up, _dp,
                                      _up, _up]
            L.orc_knn_dk.argtypes = [_dp, _u64, _u64, _dp, _up, _u64, _u64, _u64, _up, _dp, _up,
                                     _up]
            L.orc_epsnn_dk.argtypes = [_dp, _u64, _u64, _dp, _up, _u64, C.c_double, _u64, _up,
                                       _dp, _up, _up]
            L.orc_dtw_all.argtypes = [_dp, _u64, _u64, _dp, _up, _u64, _u64, _dp]
            L.orc_dk_all.argtypes = [_dp, _u64, _u64, _dp, _up, _u64, _dp]
            L.orc_knn_dk_sub.argtypes = [_dp, _u64, _u64, _dp, _up, _u64, _u64, _u64, _up, _dp,
                                         _up, _up]
            L.orc_dk_sub_full.argtypes = [_dp, _u64, _dp, _u64, _u64, _dp, _up]
        getattr(L, p + "envelope").argtypes = [_dp, _u64, _u64, _u64, _dp, _dp]
        getattr(L, p + "lb_box").argtypes = [_dp, _dp, _u64, _u64, _u64, _dp]
        getattr(L, p + "lb_sigma_min").argtypes = [_dp, _dp, _u64, _u64, _u64, _dp]
        getattr(L, p + "dtw_banded").argtypes = [_dp, _u64, _dp, _u64, _u64, _u64, _dp]
        getattr(L, p + "dtw_early_abandon").argtypes = [_dp, _u64, _dp, _u64, _u64, _u64,
                                                        C.c_double, _ip, _dp]
        getattr(L, p + "dk_full").argtypes = [_dp, _u64, _dp, _u64, _u64, _dp]
        getattr(L, p + "gdk").argtypes = [_dp, _u64, _dp, _u64, _u64, C.c_double, _dp]
        getattr(L, p + "sparse_dk").argtypes = [_dp, _u64, _dp, _u64, _u64, C.c_double, _ip, _dp]
        getattr(L, p + "znormalize").argtypes = [_dp, _u64, _u64, _dp]
        getattr(L, p + "gdk_sub").argtypes = [_dp, _u64, _dp, _u64, _u64, C.c_double, _dp, _up]
        for f in ("sparse_dk_sub", "sub_search_dk"):
            getattr(L, p + f).argtypes = [_dp, _u64, _dp, _u64, _u64, C.c_double, _ip, _dp, _up]

    # -- helpers --------------------------------------------------------------------------
    def _call(self, name, *args):
        rc = getattr(self.lib, self.p + name)(*args)
        if rc != 0:
            msg = self.lib.ref_last_error().decode() if self.kind == "reference" else name
            if rc == 1:
                raise ValueError(msg)
            raise OracleError(f"{name}: rc={rc} {msg}")

    @staticmethod
    def _s(x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x.reshape(-1, 1)
        return x

    # -- primitives -----------------------------------------------------------------------
    def envelope(self, t, r):
        t = self._s(t)
        lo = np.empty_like(t)
        hi = np.empty_like(t)
        self._call("envelope", _dptr(t), t.shape[0], t.shape[1], r, _dptr(lo), _dptr(hi))
        return lo, hi

    def lb_box(self, cand, query, r):
        c, q = self._s(cand), self._s(query)
        out = np.zeros(1)
        self._call("lb_box", _dptr(c), _dptr(q), c.shape[0], c.shape[1], r, _dptr(out))
        return float(out[0])

    def lb_sigma_min(self, s, t, r):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        self._call("lb_sigma_min", _dptr(s), _dptr(t), s.shape[0], s.shape[1], r, _dptr(out))
        return float(out[0])

    def dtw_banded(self, s, t, r):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        self._call("dtw_banded", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1], r,
                   _dptr(out))
        return float(out[0])

    def dtw_early_abandon(self, s, t, r, eps):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        ex = C.c_int(0)
        self._call("dtw_early_abandon", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1],
                   r, eps, C.byref(ex), _dptr(out))
        return bool(ex.value), float(out[0])

    def dk_full(self, s, t):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        self._call("dk_full", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1], _dptr(out))
        return float(out[0])

    def gdk(self, s, t, eps=float("inf")):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        self._call("gdk", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1], eps, _dptr(out))
        return float(out[0])

    def sparse_dk(self, s, t, eps):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        ex = C.c_int(0)
        self._call("sparse_dk", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1], eps,
                   C.byref(ex), _dptr(out))
        return bool(ex.value), float(out[0])

    def gdk_sub(self, s, t, eps=float("inf")):
        """-> (distance, end_index): SubMatch of gdk_sub (dogkeeper.cpp:96-111)."""
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        end = np.zeros(1, dtype=np.uint64)
        self._call("gdk_sub", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1], eps,
                   _dptr(out), _uptr(end))
        return float(out[0]), int(end[0])

    def _sub(self, name, s, t, eps):
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        end = np.zeros(1, dtype=np.uint64)
        found = C.c_int(0)
        self._call(name, _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1], eps,
                   C.byref(found), _dptr(out), _uptr(end))
        return (float(out[0]), int(end[0])) if found.value else None

    def sparse_dk_sub(self, s, t, eps):
        """-> (distance, end_index) or None (std::nullopt), dogkeeper.cpp:235-241."""
        return self._sub("sparse_dk_sub", s, t, eps)

    def sub_search_dk(self, s, t, eps=float("inf")):
        """-> (distance, end_index) or None, search.cpp:241-248."""
        return self._sub("sub_search_dk", s, t, eps)

    def dk_sub_full(self, s, t):
        """Brute-force subsequence DK (port only) -> (distance, end_index)."""
        assert self.kind == "port"
        s, t = self._s(s), self._s(t)
        out = np.zeros(1)
        end = np.zeros(1, dtype=np.uint64)
        self._call("dk_sub_full", _dptr(s), s.shape[0], _dptr(t), t.shape[0], s.shape[1],
                   _dptr(out), _uptr(end))
        return float(out[0]), int(end[0])

    def znormalize(self, s):
        s = self._s(s)
        out = np.empty_like(s)
        self._call("znormalize", _dptr(s), s.shape[0], s.shape[1], _dptr(out))
        return out

    # -- drivers ------------------------------------------------------------------------
    def knn(self, query, data: Dataset, k: int, metric: str, r: int = 0, threads: int = 1):
        """-> (indices u64[], distances f64[], counters u64[5])"""
        q = self._s(query)
        cap = max(1, min(k, data.n))
        idx = np.zeros(cap, dtype=np.uint64)
        dist = np.zeros(cap)
        cnt = np.zeros(1, dtype=np.uint64)
        ctr = np.zeros(5, dtype=np.uint64)
        if self.kind == "reference":
            h = data.ref_handle(self.lib)
            self._call("knn", h, _dptr(q), q.shape[0], q.shape[1], _METRIC[metric],
                       k, r, threads, cap, _uptr(idx), _dptr(dist), _uptr(cnt), _uptr(ctr), None)
        elif metric == "dtw":
            self._call("knn_dtw", _dptr(q), q.shape[0], q.shape[1], _dptr(data.values),
                       _uptr(data.lengths), data.n, k, r, cap, _uptr(idx), _dptr(dist),
                       _uptr(cnt), _uptr(ctr))
        elif metric == "dk_sub":
            self._call("knn_dk_sub", _dptr(q), q.shape[0], q.shape[1], _dptr(data.values),
                       _uptr(data.lengths), data.n, k, cap, _uptr(idx), _dptr(dist), _uptr(cnt),
                       _uptr(ctr))
        else:
            self._call("knn_dk", _dptr(q), q.shape[0], q.shape[1], _dptr(data.values),
                       _uptr(data.lengths), data.n, k, cap, _uptr(idx), _dptr(dist), _uptr(cnt),
                       _uptr(ctr))
        n = int(cnt[0])
        return idx[:n].copy(), dist[:n].copy(), ctr

    def knn_batch(self, queries: np.ndarray, data: Dataset, k: int, metric: str, r: int = 0,
                  threads: int = 0):
        """Query-parallel batch (reference lib only): queries [nq, L, d]."""
        assert self.kind == "reference"
        qs = np.ascontiguousarray(queries, dtype=np.float64)
        nq, L, d = qs.shape
        cap = max(1, min(k, data.n))
        idx = np.zeros((nq, cap), dtype=np.uint64)
        dist = np.zeros((nq, cap))
        cnt = np.zeros(nq, dtype=np.uint64)
        ctr = np.zeros((nq, 5), dtype=np.uint64)
        h = data.ref_handle(self.lib)
        threads = threads or os.cpu_count() or 1
        self._call("knn_batch", h, _dptr(qs), nq, L, d, _METRIC[metric], k, r, threads,
                   cap, _uptr(idx), _dptr(dist), _uptr(cnt), _uptr(ctr))
        return idx, dist, cnt, ctr

    def epsnn_dk(self, query, data: Dataset, eps: float):
        q = self._s(query)
        cap = max(1, data.n)
        idx = np.zeros(cap, dtype=np.uint64)
        dist = np.zeros(cap)
        cnt = np.zeros(1, dtype=np.uint64)
        ctr = np.zeros(5, dtype=np.uint64)
        if self.kind == "reference":
            h = data.ref_handle(self.lib)
            self._call("epsnn_dk", h, _dptr(q), q.shape[0], q.shape[1], eps, 1, cap, _uptr(idx),
                       _dptr(dist), _uptr(cnt), _uptr(ctr))
        else:
            self._call("epsnn_dk", _dptr(q), q.shape[0], q.shape[1], _dptr(data.values),
                       _uptr(data.lengths), data.n, eps, cap, _uptr(idx), _dptr(dist), _uptr(cnt),
                       _uptr(ctr))
        n = int(cnt[0])
        return idx[:n].copy(), dist[:n].copy(), ctr

    # brute-force all-candidate distances (port only)
    def dtw_all(self, query, data: Dataset, r: int):
        assert self.kind == "port"
        q = self._s(query)
        out = np.zeros(data.n)
        self._call("dtw_all", _dptr(q), q.shape[0], q.shape[1], _dptr(data.values),
                   _uptr(data.lengths), data.n, r, _dptr(out))
        return out

    def dk_all(self, query, data: Dataset):
        assert self.kind == "port"
        q = self._s(query)
        out = np.zeros(data.n)
        self._call("dk_all", _dptr(q), q.shape[0], q.shape[1], _dptr(data.values),
                   _uptr(data.lengths), data.n, _dptr(out))
        return out


_synth_lib = None


def _synth():
    """The config generator built into oracle/_build (bench.py's reference arm: no product .so)."""
    global _synth_lib
    with _lock:
        if _synth_lib is None:
            if not os.path.exists(SYNTH_SO):
                subprocess.run(["make", "-s", "-C", HERE, "synth"], check=True)
            L = C.CDLL(SYNTH_SO)
            L.tsw_synth_shape.argtypes = [C.c_int, C.c_int, _up, _up, _up, _up, _up]
            L.tsw_synth_generate.argtypes = [C.c_int, C.c_int, _u64, _dp, C.POINTER(C.c_int32)]
            _synth_lib = L
        return _synth_lib


def synth_shape(config: int, part: int = 0) -> dict:
    vals = [_u64() for _ in range(5)]
    if _synth().tsw_synth_shape(config, part, *[C.byref(v) for v in vals]) != 0:
        raise ValueError(f"unknown config {config}")
    return dict(zip(["count", "len", "d", "r", "k"], [v.value for v in vals]))


def synth(config: int, part: int, seed: int = 20181127):
    """-> (values f64[count, len, d], labels i32[count]); same bytes as the product's synth."""
    sh = synth_shape(config, part)
    out = np.empty((sh["count"], sh["len"], sh["d"]), dtype=np.float64)
    lab = np.empty(sh["count"], dtype=np.int32)
    if _synth().tsw_synth_generate(config, part, seed, _dptr(out),
                                   lab.ctypes.data_as(C.POINTER(C.c_int32))) != 0:
        raise ValueError(f"synth({config}, {part}) failed")
    return out, lab


def port() -> Oracle:
    with _lock:
        if "port" not in _cache:
            if not os.path.exists(PORT_SO):
                build(ref=False)
            _cache["port"] = Oracle(PORT_SO, "port")
        return _cache["port"]


def ref() -> Oracle:
    with _lock:
        if "ref" not in _cache:
            if not os.path.exists(REF_SO):
                if not os.path.isdir(REF_ROOT):
                    raise OracleError("oracle/_ref not built and /root/reference absent")
                build(ref=True)
            _cache["ref"] = Oracle(REF_SO, "reference")
        return _cache["ref"]


class RefIO:
    """The reference's own load_dataset / save_dataset (oracle/_ref/libtswarp_ref_io.so, built
    against nlohmann/json 3.11.3).  load() -> (values f64[total*d], lengths u64[n], d, labels |
    None, meta dict) or raises (kind, message) as RefIOError."""

    ERR = {1: "invalid_argument", 3: "runtime_error", 4: "ValidationError", 5: "ParseError",
           6: "IoError"}

    def __init__(self, path: str):
        L = self.lib = C.CDLL(path)
        L.refio_last_error.restype = C.c_char_p
        L.refio_load.restype = C.c_void_p
        L.refio_load.argtypes = [C.c_char_p, _ip]
        L.refio_free.argtypes = [C.c_void_p]
        L.refio_shape.argtypes = [C.c_void_p, _up, _up, _up, _ip, _up]
        L.refio_copy.argtypes = [C.c_void_p, _dp, _up]
        L.refio_label.argtypes = [C.c_void_p, _u64]
        L.refio_label.restype = C.c_char_p
        L.refio_meta.argtypes = [C.c_void_p, _u64, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]
        L.refio_save.argtypes = [C.c_void_p, C.c_char_p]

    def _open(self, path):
        rc = C.c_int(0)
        h = self.lib.refio_load(os.fsencode(path), C.byref(rc))
        if not h:
            raise RefIOError(self.ERR.get(rc.value, str(rc.value)),
                             self.lib.refio_last_error().decode("utf-8", "replace"))
        return h

    def load(self, path):
        h = self._open(path)
        try:
            n, d, tot, nm = (np.zeros(1, dtype=np.uint64) for _ in range(4))
            lab = C.c_int(0)
            self.lib.refio_shape(h, _uptr(n), _uptr(d), _uptr(tot), C.byref(lab), _uptr(nm))
            n, d, tot, nm = int(n[0]), int(d[0]), int(tot[0]), int(nm[0])
            vals = np.zeros(tot * d)
            lens = np.zeros(n, dtype=np.uint64)
            self.lib.refio_copy(h, _dptr(vals), _uptr(lens))
            labels = [self.lib.refio_label(h, i).decode("utf-8") for i in range(n)] if lab.value else None
            meta = {}
            for i in range(nm):
                k, v = C.c_char_p(), C.c_char_p()
                self.lib.refio_meta(h, i, C.byref(k), C.byref(v))
                meta[k.value.decode("utf-8")] = v.value.decode("utf-8")
            return vals, lens, d, labels, meta
        finally:
            self.lib.refio_free(h)

    def resave(self, src, dst):
        """load_dataset(src) then save_dataset(dst) through the reference."""
        h = self._open(src)
        try:
            if self.lib.refio_save(h, os.fsencode(dst)) != 0:
                raise RefIOError("save", self.lib.refio_last_error().decode())
        finally:
            self.lib.refio_free(h)


class RefIOError(Exception):
    def __init__(self, kind, message):
        super().__init__(f"{kind}: {message}")
        self.kind, self.message = kind, message


def ref_io() -> RefIO:
    with _lock:
        if "ref_io" not in _cache:
            if not os.path.exists(REF_IO_SO):
                if os.path.isdir(REF_ROOT):
                    subprocess.run(["make", "-s", "-C", HERE, "ref_io"], check=True)
                if not os.path.exists(REF_IO_SO):
                    raise OracleError("oracle/_ref/libtswarp_ref_io.so unavailable")
            _cache["ref_io"] = RefIO(REF_IO_SO)
        return _cache["ref_io"]
