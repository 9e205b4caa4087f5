"""Test-only CPU implementation of the ShardEngine primitives.

Used by the multi-rank gloo tests to drive the PRODUCT's IHT loop
(paper_1608_01398_b200.iht) and its sharding logic (engine.ShardEngine:
global/local indices, all-reduced partial products, top-k candidate merge)
on CPU ranks.  The per-shard arithmetic comes from the oracle (oracle/), so
this is test infrastructure, never a product fallback.
"""
import numpy as np
import torch

import oracle
from paper_1608_01398_b200.engine import Genotypes, ShardEngine


class OracleShard:
    """Columns [j0, j0 + p_local) of an oracle matrix, as an engine operand."""

    def __init__(self, full: "oracle.OraclePacked", j0: int, j1: int):
        self.n = full.n
        self.p = j1 - j0
        self.mat = oracle.OraclePacked(n=full.n, p=self.p, data=full.data[j0:j1].copy(),
                                       u=full.u[j0:j1].copy(), v=full.v[j0:j1].copy())


class CpuEngine(ShardEngine):
    def __init__(self, geno: Genotypes, y, cov, kmax):
        super().__init__(geno, 0 if cov is None else cov.shape[1], kmax)
        self.mat = geno.matrix.mat
        self.y = np.asarray(y, dtype=np.float64)
        self.C = None if cov is None else np.asarray(cov, dtype=np.float64)
        self.bufs = {"fit": torch.zeros(self.n, dtype=torch.float64),
                     "img": torch.zeros(self.n, dtype=torch.float64)}
        self.beta = np.zeros(self.p)
        self.g = np.zeros(self.p)
        self.r = np.zeros(self.n)

    def _buffer(self, which):
        return self.bufs[which]

    def _ax_partial(self, which, idx_l, w_l):
        self.bufs[which].copy_(torch.from_numpy(self.mat.ax_columns(idx_l, w_l)))
        self.kernel_launches += 1

    def _scatter_beta(self, idx_l, vals):
        self.beta[idx_l] = vals

    def reset_beta(self):
        self.beta[:] = 0.0

    def _finish_refresh(self, bcov, has_fit, sup_l):
        fit = self.bufs["fit"].numpy().copy() if has_fit else np.zeros(self.n)
        if self.c:
            fit = fit + self.C @ np.asarray(bcov, dtype=np.float64)
        self.r = self.y - fit
        loss = 0.5 * float(self.r @ self.r)
        self.g = -self.mat.aty_genetic(self.r)
        gcov = -(self.C.T @ self.r) if self.c else np.zeros(0)
        gmax = float(np.abs(self.g).max()) if self.p else 0.0
        return loss, gmax, gcov, self.g[sup_l].copy()

    def _finish_image(self, wcov):
        img = self.bufs["img"].numpy().copy()
        if wcov is not None and self.c:
            img = img + self.C @ np.asarray(wcov, dtype=np.float64)
        return float(img @ img)

    def _topk_local(self, mode, mu, k):
        vals = self.g.copy() if mode == 0 else self.beta - mu * self.g
        keys = np.abs(vals).view(np.uint64) + np.uint64(1)
        gidx = np.arange(self.p, dtype=np.int64) + self.geno.j_base
        order = np.lexsort((gidx, ~keys))[:k]
        return keys[order], gidx[order], vals[order]

    def gradient(self):
        return self.g.copy()

    def residuals(self):
        return self.r.copy()
