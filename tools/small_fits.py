"""A few resident native fits at config 1 or 2 (for ncu launch lists of the small kernels)."""
import sys

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

n, p, k = {"c1": (1000, 10000, 10), "c2": (5000, 100000, 20),
           "c3s8": (100000, 125000, 20)}[sys.argv[1]]  # c3s8: one GPU's shard of config 3 on 8
m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=k, seed=1398))
cfg = gi.IhtConfig(k=k)
gi.fit(view, y, cfg)
for _ in range(3):
    r = gi.fit(view, y, cfg, _resident=True)
print("iterations", r.iterations)
