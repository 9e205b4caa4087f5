import numpy as np
import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype
m = gi.PackedGenotypeMatrix.synthetic(1000, 10000, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=1000))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=10, seed=1398))
for _ in range(5):
    r = gi.fit(view, y, gi.IhtConfig(k=10))
print(r.iterations)
