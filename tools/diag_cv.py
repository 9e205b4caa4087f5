"""Replay one stress_cv case fold by fold: device fold fits (compact training
copies, the cv_iht path) vs the oracle's per-fold fits."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import stress_cv  # noqa: E402,F401  (sets up sys.path)
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402
from paper_1608_01398_b200 import model_select as ms  # noqa: E402

seed = int(sys.argv[1])
rng = np.random.default_rng(seed)
n = int(rng.integers(150, 1500))
p = int(rng.integers(50, 3000))
miss = float(rng.choice([0.0, 0.02]))
codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
q = int(rng.integers(3, 6))
path = np.arange(1, int(rng.integers(3, 11)))
std_mode = str(rng.choice(["train", "global"]))
warm = bool(rng.random() < 0.3)
covar = rng.standard_normal((n, 2)) if rng.random() < 0.3 else None
support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 6))), replace=False))
ref_p = oracle.OraclePacked.from_codes(codes)
y = ref_p.ax_columns(support, rng.standard_normal(support.size)) \
    + rng.normal(0, float(rng.choice([0.1, 0.5])), n)
block = gi.CovariateBlock.build(covar, n=n)
view = gi.StandardizedView(gi.PackedGenotypeMatrix.from_codes(codes), block)
plan = gi.CvPlan.build(n, q, path, seed=seed)
want = oracle.cv(oracle.OracleView(ref_p, block.values), y, q, path, seed, std_mode=std_mode,
                 warm_start=warm, labels=plan.fold_labels)
labels = plan.fold_labels
for f in range(q):
    test, train = np.flatnonzero(labels == f), np.flatnonzero(labels != f)
    v_tr, _ = ms._fold_views(view, train, test, std_mode, compact=True)
    wm = None
    for ki, k in enumerate(path):
        res = gi.fit(v_tr, y[train], gi.IhtConfig(k=int(k)), warm=wm if warm else None)
        wm = res.model
        o = want.fold_fits[f][ki]
        same = np.array_equal(res.model.support, o.support) and res.iterations == o.iterations
        d = np.max(np.abs(res.model.weights - o.weights)) / np.max(np.abs(o.weights)) \
            if same and o.weights.size else np.nan
        print(f"fold {f} k={k}: device it={res.iterations} bt={res.backtracks} "
              f"oracle it={o.iterations} bt={o.backtracks} support equal "
              f"{np.array_equal(res.model.support, o.support)} beta {d:.1e}", flush=True)
