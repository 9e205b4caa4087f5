"""Config-4 CV with the covariate least squares via the cached pinv vs np.linalg.lstsq."""
import time

import numpy as np
import torch

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.geno_matrix import CovariateBlock
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

n, p = 20000, 500000
m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=10, seed=1398))
plan = gi.CvPlan.build(n, 5, np.arange(1, 21), seed=2016)
orig = CovariateBlock.least_squares


def via_lstsq(self, yy):
    return np.linalg.lstsq(self.values, yy, rcond=None)[0]


for name, fn in (("pinv", orig), ("lstsq", via_lstsq), ("pinv", orig), ("lstsq", via_lstsq)):
    CovariateBlock.least_squares = fn
    gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gi.cv_iht(view, y, plan, gi.IhtConfig(k=20))
    torch.cuda.synchronize()
    print(f"{name}: cv_iht {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
