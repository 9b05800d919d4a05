"""tswarp_b200: a B200-native k-NN query engine for multi-dimensional time series.

The hot path of arXiv 1811.11076's reference library (`tswarp`, proj/core) -- the k-NN linear
scan under banded DTW with LB_Box pruning, and the dog-keeper (discrete Frechet) k-NN --
re-built as hand-written sm_100a CUDA kernels behind a C ABI (include/tswarp_b200.h), with a
C++ drop-in header (include/tswarp_b200.hpp) and this Python mirror (tswarp.py).
"""
from .tswarp import (  # noqa: F401
    NO_NEIGHBOR, Dataset, IoError, Neighbor, ParseError, Plan, SearchCounters, SearchReport, Store, SubMatch,
    TswError, ValidationError, device_count, dist_all, envelope, epsnn_dk, fp64_peak, knn, knn_dk,
    load_dataset, loo_accuracy, pruning_power, save_dataset, speedup,
    knn_dk_sub, knn_dtw, l2_flush, lb_box_exact_all, last_transfer_bytes, lb_box_all, lib, sparse_dk_sub,
    sub_dk_all, sub_search_dk, synth, synth_shape,
)

__all__ = [
    "NO_NEIGHBOR", "Dataset", "IoError", "Neighbor", "ParseError", "Plan", "load_dataset", "save_dataset",
    "loo_accuracy", "pruning_power", "speedup", "SearchCounters", "SearchReport", "Store", "SubMatch",
    "TswError", "ValidationError", "device_count", "dist_all", "envelope", "epsnn_dk",
    "fp64_peak", "knn", "knn_dk", "knn_dk_sub", "knn_dtw", "l2_flush", "last_transfer_bytes",
    "lb_box_all", "lb_box_exact_all", "lib", "sparse_dk_sub", "sub_dk_all", "sub_search_dk", "synth", "synth_shape",
]
