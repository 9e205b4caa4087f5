"""Small end-to-end exercise of every kernel, for compute-sanitizer runs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402

for n, p, miss in [(1030, 700, 0.05), (513, 65, 0.0)]:
    codes = oracle.random_codes(n, p, seed=n, missing_rate=miss)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    r = np.random.default_rng(1).standard_normal(n)
    a = m.aty_genetic(r)
    b = m.aty_genetic(r, mode="fast")
    m.ax_columns(np.arange(0, p, 7), np.ones(len(range(0, p, 7))))
    m.decompress(np.arange(5))
    m.subset_rows(np.arange(0, n, 3))
    m.subset_rows(np.random.default_rng(2).permutation(n)[: n // 2])  # global-load gather
    m.aty_batched(np.stack([r, -r]), mode="fast")
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=n))
    y = m.ax_columns(np.array([1, 5, 9]), np.array([1.0, -1.0, 0.5])) + r * 0.1
    f1 = gi.fit(view, y, gi.IhtConfig(k=5))
    f2 = gi.fit(view, y, gi.IhtConfig(k=5), native=False)
    assert np.array_equal(f1.model.support, f2.model.support)
    plan = gi.CvPlan.build(n, 3, np.arange(1, 4), seed=1)
    for compact in ("0", "1"):
        os.environ["GI_CV_COMPACT"] = compact
        gi.cv_iht(view, y, plan, gi.IhtConfig(k=3))
    big = gi.PackedGenotypeMatrix.synthetic(3000, 70000, 5, missing_rate=0.01)  # top-k: 18 chunks
    bview = gi.StandardizedView(big, gi.CovariateBlock.build(np.ones((3000, 10)), n=3000))
    gi.fit(bview, big.ax_columns(np.array([3, 40000]), np.array([1.0, 1.0])), gi.IhtConfig(k=40))
print("sanitize case ok")
