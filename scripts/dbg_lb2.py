import numpy as np, sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from test_gpu_parity import walks
import paper_1811_11076_b200 as tsw
rng = np.random.default_rng(8)
n = int(rng.integers(1, 200)); L = int(rng.integers(1, 64)); d = int(rng.integers(1, 5))
r = int(rng.integers(0, max(1, L // 3) + 1)); k = int(rng.integers(1, 12))
X = walks(rng, n, L, d); Q = walks(rng, 3, L, d)
gi, gd, gc = tsw.knn(tsw.Dataset(X), Q, k, "dtw", r)
print(gi, gd, gc)
