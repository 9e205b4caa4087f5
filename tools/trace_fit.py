"""Sync count / wait time of the native loop (GI_TRACE_FIT=1) at small configs."""
import os
import time

import numpy as np

os.environ["GI_TRACE_FIT"] = "1"
import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

for n, p, k in [(1000, 10000, 10), (5000, 100000, 20)]:
    m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    y, _ = simulate_phenotype(view, SimulationSpec(k_true=k, seed=1398))
    cfg = gi.IhtConfig(k=k)
    gi.fit(view, y, cfg)
    for _ in range(20):
        gi.fit(view, y, cfg, _resident=True)
    t0 = time.perf_counter()
    gi.fit(view, y, cfg, _resident=True)
    print(f"n={n} p={p}: fit {1e6 * (time.perf_counter() - t0):.0f} us", flush=True)
