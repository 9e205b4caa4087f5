"""Device time of the exact (reference-order fp64) vs fast X^T r kernels by size."""
import time

import numpy as np
import torch

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200 import _native

for n, p in [(62, 3886), (1000, 10000), (2000, 20000), (5000, 100000), (20000, 100000),
             (100000, 100000)]:
    m = gi.PackedGenotypeMatrix.synthetic(n, p, 7)
    r = np.random.default_rng(1).standard_normal(n)
    out = {}
    for mode in ("exact", "fast"):
        for _ in range(3):
            m.aty_genetic(r, mode=mode)
        t0 = time.perf_counter()
        for _ in range(10):
            m.aty_genetic(r, mode=mode)
        out[mode] = (time.perf_counter() - t0) / 10 * 1e3
    print(f"n={n:6d} p={p:6d} packed={n * p / 4e6:8.1f} MB: exact {out['exact']:8.3f} ms  "
          f"fast {out['fast']:8.3f} ms (host call incl. copies)", flush=True)
