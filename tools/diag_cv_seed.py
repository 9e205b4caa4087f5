import os, sys
import numpy as np
ROOT = "/root/repo"
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle
import paper_1608_01398_b200 as gi
from paper_1608_01398_b200 import model_select as ms
import stress_cv

def run(seed, patch=None, drop_heldout=False):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(150, 1500)); p = int(rng.integers(50, 3000))
    miss = float(rng.choice([0.0, 0.02]))
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    q = int(rng.integers(3, 6)); path = np.arange(1, int(rng.integers(3, 11)))
    std_mode = str(rng.choice(["train", "global"])); warm = bool(rng.random() < 0.3)
    covar = rng.standard_normal((n, 2)) if rng.random() < 0.3 else None
    support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 6))), replace=False))
    ref_p = oracle.OraclePacked.from_codes(codes)
    y = ref_p.ax_columns(support, rng.standard_normal(support.size)) + rng.normal(0, float(rng.choice([0.1, 0.5])), n)
    block = gi.CovariateBlock.build(covar, n=n)
    view = gi.StandardizedView(gi.PackedGenotypeMatrix.from_codes(codes), block)
    plan = gi.CvPlan.build(n, q, path, seed=seed)
    want = oracle.cv(oracle.OracleView(ref_p, block.values), y, q, path, seed, std_mode=std_mode, warm_start=warm, labels=plan.fold_labels)
    orig = ms.last_native_fit_info
    orig_ni = ms.native_inputs
    from paper_1608_01398_b200 import iht as _iht
    orig_fit = ms.fit
    if patch: ms.last_native_fit_info = lambda: None
    if drop_heldout:
        ms.native_inputs = lambda v, y, t, h=None: orig_ni(v, y, t, None)
        ms.fit = lambda *a, **k: orig_fit(*a, **{**k, "_heldout": None})
    got = gi.cv_iht(view, y, plan, gi.IhtConfig(k=int(path.max())), std_mode=std_mode, warm_start=warm)
    ms.last_native_fit_info = orig
    ms.native_inputs = orig_ni
    ms.fit = orig_fit
    print(seed, "drop" if drop_heldout else ("patch" if patch else "heldout"), "k_best", got.k_best, want.k_best)
    print(" got mse", got.mse.ravel()[:12])
    print(" want   ", want.mse.ravel()[:12])
    print(" rel max", np.max(np.abs(got.mse - want.mse)) / np.max(np.abs(want.mse)))

for s in (142020, 142055):
    run(s, drop_heldout=True)
