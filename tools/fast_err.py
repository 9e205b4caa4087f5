"""Error of the fast X^T r against the exact kernel, relative to rms(g)."""
import numpy as np

import paper_1608_01398_b200 as gi
import oracle

rng = np.random.default_rng(3)
for n, p, miss in [(100, 500, 0.0), (1000, 4000, 0.05), (20000, 20000, 0.02), (100000, 4000, 0.0)]:
    codes = oracle.random_codes(n, p, seed=n, missing_rate=miss)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    worst = 0.0
    for _ in range(5):
        r = rng.standard_normal(n) * rng.choice([1.0, 1e-3, 1e3])
        r[rng.integers(0, n)] *= 30.0  # an outlier
        ex = m.aty_genetic(r, mode="exact")
        fa = m.aty_genetic(r, mode="fast")
        worst = max(worst, np.max(np.abs(fa - ex)) / np.sqrt(np.mean(ex ** 2)))
    print(f"n={n} p={p} miss={miss}: max |fast - exact| / rms = {worst:.2e}", flush=True)
