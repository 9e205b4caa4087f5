"""Where config-4 CV time goes: fold construction, masked vs compact fold fits."""
import os
import time

import numpy as np
import torch

import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.model_select import FoldGenotypes
from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

n, p = 20000, 500000
m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
y, _ = simulate_phenotype(view, SimulationSpec(k_true=10, seed=1398))
plan = gi.CvPlan.build(n, 5, np.arange(1, 21), seed=2016)
train = np.flatnonzero(plan.fold_labels != 0)


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) / reps * 1e3:9.2f} ms", flush=True)
    return out


keep = np.zeros(n, np.uint8)
keep[train] = 1
u, v = t("masked_stats", lambda: m.masked_stats(keep))
sub = t("subset_rows", lambda: m.subset_rows(train))
t("subset_rows + with_stats", lambda: m.subset_rows(train).with_stats(u, v))
fold_m = m.with_stats(u, v)
masked = gi.StandardizedView(FoldGenotypes(fold_m, train), view.covariates.subset_rows(train))
compact = gi.StandardizedView(sub.with_stats(u, v), view.covariates.subset_rows(train))
for k in (5, 10, 20):
    a = t(f"fit masked k={k}", lambda: gi.fit(masked, y[train], gi.IhtConfig(k=k)))
    b = t(f"fit compact k={k}", lambda: gi.fit(compact, y[train], gi.IhtConfig(k=k)))
    print("   iterations", a.iterations, b.iterations, "aty ms/launch",
          flush=True)
for c in ("0", "1"):
    os.environ["GI_CV_COMPACT"] = c
    t(f"cv_iht compact={c}", lambda: gi.cv_iht(view, y, plan, gi.IhtConfig(k=20)), reps=2)
