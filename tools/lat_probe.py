"""Per-fit and per-iteration host latency of the native loop at small configs."""
import sys
import time

import numpy as np

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

for n, p, k in [(1000, 10000, 10), (5000, 100000, 20)]:
    m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    y, _ = simulate_phenotype(view, SimulationSpec(k_true=k, seed=1398))
    for mi in (1, 2, 4, 8, 200):
        cfg = gi.IhtConfig(k=k, max_iter=mi)
        for _ in range(5):
            gi.fit(view, y, cfg)
        ts, its = [], 0
        for _ in range(40):
            t0 = time.perf_counter()
            r = gi.fit(view, y, cfg)
            ts.append(time.perf_counter() - t0)
            its = r.iterations
        ts2 = []
        for _ in range(40):
            t0 = time.perf_counter()
            r = gi.fit(view, y, cfg, _resident=True)
            ts2.append(time.perf_counter() - t0)
        print(f"n={n} p={p} k={k} max_iter={mi:3d}: iters={its:2d} fit {np.median(ts)*1e6:8.0f} us"
              f"  resident {np.median(ts2)*1e6:8.0f} us", flush=True)
