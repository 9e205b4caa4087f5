"""World-size-2 (gloo, CPU) runs of the product's sharded IHT loop.

Each rank owns a contiguous SNP block (dist.shard_range) and runs
paper_1608_01398_b200.iht.fit; the engine's sharding logic all-reduces the
n-length partial products and merges per-rank top-k candidate lists.  The
per-shard arithmetic is the oracle's (tests/cpu_engine.py), so the sharded
fit must reproduce the unsharded oracle fit: identical support and iteration
count, weights and losses to 1e-9 (only the all-reduce summation order differs).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(seed):
    rng = np.random.default_rng(seed)
    n, p = 300, 777
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=0.03)
    full = oracle.OraclePacked.from_codes(codes)
    support = np.sort(rng.choice(p, 6, replace=False))
    y = full.ax_columns(support, rng.normal(0, 1, 6)) + rng.normal(0, 0.3, n)
    return full, y


class _View:
    def __init__(self, n, p, cov):
        from paper_1608_01398_b200 import CovariateBlock, StandardizedView  # noqa: F401
        self.n, self.p = n, p
        self.covariates = None if cov is None else type("B", (), {"values": cov, "c": cov.shape[1]})
        self.c = 0 if cov is None else cov.shape[1]
        self.genotypes = self


def _worker(rank, world, port, seed, k, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import cpu_engine
        from paper_1608_01398_b200 import IhtConfig, fit
        from paper_1608_01398_b200.dist import TorchComm, shard_range
        from paper_1608_01398_b200.engine import Genotypes

        full, y = _case(seed)
        cov = oracle.intercept(full.n)
        comm = TorchComm()
        j0, j1 = shard_range(full.p, world, rank)
        geno = Genotypes(cpu_engine.OracleShard(full, j0, j1), j_base=j0, p_global=full.p,
                         comm=comm)
        eng = cpu_engine.CpuEngine(geno, y, cov, kmax=k)
        res = fit(_View(full.n, full.p, cov), y, IhtConfig(k=k), engine=eng)
        out_q.put((rank, res.model.support, res.model.weights, res.model.covar,
                   res.loss_trace, res.iterations, res.reason))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,k", [(11, 6), (12, 3), (13, 10)])
def test_sharded_fit_matches_unsharded_oracle(seed, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, k, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    full, y = _case(seed)
    want = oracle.fit(oracle.OracleView(full, oracle.intercept(full.n)), y, k)
    for rank, support, weights, covar, trace, iters, reason in results:
        np.testing.assert_array_equal(support, want.support)
        assert iters == want.iterations and reason == want.reason
        np.testing.assert_allclose(weights, want.weights, rtol=1e-9)
        np.testing.assert_allclose(covar, want.covar, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(trace, want.loss_trace, rtol=1e-9)
    # every rank took identical decisions
    np.testing.assert_array_equal(results[0][1], results[1][1])
