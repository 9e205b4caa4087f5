"""Replay stress cases with the covariate init from the cached pinv vs exact lstsq."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import stress_parity as sp  # noqa: E402
from paper_1608_01398_b200.geno_matrix import CovariateBlock  # noqa: E402

orig = CovariateBlock.least_squares
for seed in [int(a) for a in sys.argv[1:]]:
    for name in ("pinv", "lstsq"):
        CovariateBlock.least_squares = orig if name == "pinv" else \
            (lambda self, y: np.linalg.lstsq(self.values, y, rcond=None)[0])
        ok, desc = sp.case(seed)
        print(name, ok, desc, flush=True)
