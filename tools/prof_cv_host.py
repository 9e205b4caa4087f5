import cProfile, pstats, sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype
m = gi.PackedGenotypeMatrix.synthetic(20000, 500000, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=20000))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=10, seed=1398))
plan = gi.CvPlan.build(20000, 5, np.arange(1, 21), seed=2016)
gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
