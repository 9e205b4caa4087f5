"""Host-side profile of device fits at a small config (where the host loop dominates)."""
import cProfile
import pstats
import sys
import time

import numpy as np

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

n, p, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=k, seed=1398))
cfg = gi.IhtConfig(k=k)
st = gi.initial_state(view, y, cfg)
for _ in range(3):
    gi.fit(view, y, cfg, engine=st.engine)
t0 = time.perf_counter()
its = 0
for _ in range(20):
    its += gi.fit(view, y, cfg, engine=st.engine).iterations
dt = time.perf_counter() - t0
print(f"{its} iterations in {dt*1e3:.1f} ms -> {its/dt:.0f} it/s, {dt/its*1e6:.0f} us/iter")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    gi.fit(view, y, cfg, engine=st.engine)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
