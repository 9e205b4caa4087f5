"""Cost split of building CV fold copies: allocation + gather + stats vs freeing."""
import gc
import time

import numpy as np
import torch

import paper_1608_01398_b200 as gi

n, p = 20000, 500000
m = gi.PackedGenotypeMatrix.synthetic(n, p, 1608)
labels = gi.CvPlan.build(n, 5, np.arange(1, 3), seed=2016).fold_labels
for rep in range(3):
    subs = []
    for f in range(5):
        rows = np.flatnonzero(labels != f)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        subs.append(m.subset_rows(rows))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        w = subs[-1].with_stats(subs[-1].u, subs[-1].v)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        del w
        gc.collect()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"rep {rep} fold {f}: subset {1e3 * (t1 - t0):7.2f} ms  with_stats "
              f"{1e3 * (t2 - t1):6.2f} ms  free(with_stats) {1e3 * (t3 - t2):6.2f} ms", flush=True)
    t0 = time.perf_counter()
    del subs
    gc.collect()
    torch.cuda.synchronize()
    print(f"rep {rep}: free 5 fold copies {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
