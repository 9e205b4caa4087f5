"""The sharded DEVICE path on one GPU: two processes, each owning a contiguous
SNP block (its own device-resident shard), joined by gloo -- through the native
sharded loop (gi_fit_sharded with host-callback collectives) and through the
Python loop over DeviceEngine.
Collectives are host-staged, so no kernel waits on another process.  The
sharded fit must reproduce the unsharded device fit and the oracle: identical
support and iteration count, weights and loss to 1e-6."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu

N, P, K, SEED = 3000, 20011, 12, 77


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, native):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1608_01398_b200 as gi
        from paper_1608_01398_b200.dist import ShardedGenotypes, TorchComm
        from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

        torch.cuda.set_device(0)
        comm = TorchComm()
        geno = ShardedGenotypes.synthetic(N, P, SEED, comm, device=0, missing_rate=0.01)
        view = gi.StandardizedView(geno, gi.CovariateBlock.build(None, n=N))
        y, truth = simulate_phenotype(view, SimulationSpec(k_true=K, seed=5))
        res = gi.fit(view, y, gi.IhtConfig(k=K), native=native)
        if native:
            assert geno.native_comm().kind == "callbacks"  # gloo: host-staged collectives
        q.put((rank, y, res.model.support, res.model.weights, res.model.covar, res.loss_trace,
               res.iterations, res.reason))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("native", [True, False], ids=["native-sharded-loop", "python-loop"])
def test_two_shards_on_one_gpu_match_single_device_fit(native):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, native)) for r in range(world)]
    for p_ in procs:
        p_.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    import paper_1608_01398_b200 as gi

    y = out[0][1]
    np.testing.assert_array_equal(out[1][1], y)
    full = gi.PackedGenotypeMatrix.synthetic(N, P, SEED, missing_rate=0.01)
    view = gi.StandardizedView(full, gi.CovariateBlock.build(None, n=N))
    want = gi.fit(view, y, gi.IhtConfig(k=K))
    ref = oracle.fit(oracle.OracleView(oracle.OraclePacked.from_bed(np.array(full.data), N),
                                       oracle.intercept(N)), y, K)
    np.testing.assert_array_equal(want.model.support, ref.support)
    assert want.iterations == ref.iterations
    for rank, _, support, weights, covar, trace, iters, reason in out:
        np.testing.assert_array_equal(support, want.model.support)
        assert iters == want.iterations and reason == want.reason
        np.testing.assert_allclose(weights, want.model.weights, rtol=1e-6)
        np.testing.assert_allclose(covar, want.model.covar, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(trace, want.loss_trace, rtol=1e-6)


def _nccl_worker(port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        import paper_1608_01398_b200 as gi
        from paper_1608_01398_b200.dist import ShardedGenotypes, TorchComm
        from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

        comm = TorchComm()
        geno = ShardedGenotypes.synthetic(N, P, SEED, comm, device=0, missing_rate=0.01)
        view = gi.StandardizedView(geno, gi.CovariateBlock.build(None, n=N))
        y, _ = simulate_phenotype(view, SimulationSpec(k_true=K, seed=5))
        out = {}
        for native in (True, False):
            res = gi.fit(view, y, gi.IhtConfig(k=K), native=native)
            out[native] = (res.model.support, res.model.weights, res.model.covar,
                           res.loss_trace, res.iterations, res.reason)
        q.put((y, out, geno.native_comm().kind))
    finally:
        dist.destroy_process_group()


def test_nccl_backend_world_one_matches_device_fit():
    """The NCCL communicator of the native sharded loop (dlopen'd libnccl,
    in-place device all-reduce, device all-gathers) on a world of one:
    gi_fit_sharded runs every exchange step through real NCCL collectives and
    must reproduce the unsharded gi_fit (to 1e-12: only the image norm's
    summation order differs)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    proc = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    proc.start()
    y, out, kind = q.get(timeout=600)
    proc.join(timeout=120)
    assert proc.exitcode == 0
    assert kind == "nccl"
    import paper_1608_01398_b200 as gi

    full = gi.PackedGenotypeMatrix.synthetic(N, P, SEED, missing_rate=0.01)
    view = gi.StandardizedView(full, gi.CovariateBlock.build(None, n=N))
    want = gi.fit(view, y, gi.IhtConfig(k=K))
    for native, (support, weights, covar, trace, iters, reason) in out.items():
        np.testing.assert_array_equal(support, want.model.support)
        assert iters == want.iterations and reason == want.reason
        if native:  # same kernels except the image norm's summation order (the
            # sharded loop all-reduces X_S w before the norm; gi_fit fuses them)
            np.testing.assert_allclose(weights, want.model.weights, rtol=1e-12, atol=0)
            np.testing.assert_allclose(trace, want.loss_trace, rtol=1e-12, atol=0)
        np.testing.assert_allclose(weights, want.model.weights, rtol=1e-6)
        np.testing.assert_allclose(covar, want.model.covar, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(trace, want.loss_trace, rtol=1e-6)


def _empty_shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1608_01398_b200 as gi
        from paper_1608_01398_b200.dist import ShardedGenotypes, TorchComm

        torch.cuda.set_device(0)
        codes = oracle.random_codes(400, 300, seed=13, missing_rate=0.02)
        j0, j1 = (0, 300) if rank == 0 else (300, 300)  # rank 1 owns no SNPs
        geno = ShardedGenotypes(gi.PackedGenotypeMatrix.from_codes(codes[:, j0:j1]), j0, 300,
                                TorchComm())
        view = gi.StandardizedView(geno, gi.CovariateBlock.build(None, n=400))
        y = oracle.OraclePacked.from_codes(codes).ax_columns(np.array([4, 99]),
                                                            np.array([1.0, -1.0]))
        res = gi.fit(view, y, gi.IhtConfig(k=3))
        q.put((rank, res.model.support, res.iterations))
    finally:
        dist.destroy_process_group()


def test_sharded_fit_with_an_empty_shard():
    """A rank that owns no SNPs still takes part in every exchange (its X^T r
    plan, top-k and gather are empty) and the fit matches the unsharded one."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_empty_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    import paper_1608_01398_b200 as gi

    codes = oracle.random_codes(400, 300, seed=13, missing_rate=0.02)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    y = oracle.OraclePacked.from_codes(codes).ax_columns(np.array([4, 99]), np.array([1.0, -1.0]))
    want = gi.fit(gi.StandardizedView(m, gi.CovariateBlock.build(None, n=400)), y,
                  gi.IhtConfig(k=3))
    for _, support, iters in out:
        np.testing.assert_array_equal(support, want.model.support)
        assert iters == want.iterations


def _path_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1608_01398_b200 as gi
        from paper_1608_01398_b200.dist import ShardedGenotypes, TorchComm
        from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

        torch.cuda.set_device(0)
        comm = TorchComm()
        # 1000 x 12000: 3 MiB of tiles globally (fast X^T r kernel), 1.5 MiB per
        # shard -- each rank alone would have picked the exact kernel
        geno = ShardedGenotypes.synthetic(1000, 12000, 31, comm, device=0)
        view = gi.StandardizedView(geno, gi.CovariateBlock.build(None, n=1000))
        y, _ = simulate_phenotype(view, SimulationSpec(k_true=8, seed=9))
        # default workers (8): the path must still run its sharded fits one at a
        # time in the same order on both ranks (one communicator per group)
        res = gi.fit_path(view, y, [3, 8, 12])
        q.put((rank, y, [(r.model.support, r.model.weights, r.loss_trace, r.iterations)
                         for r in res]))
    finally:
        dist.destroy_process_group()


def test_fit_path_on_sharded_view_matches_unsharded_path(monkeypatch):
    """fit_path over an SNP-sharded view (2 ranks, gloo callbacks, one GPU):
    its fits share the process group's communicator, so they must run
    sequentially; and the X^T r kernel is chosen on the global shape, so the
    shards (1.5 MiB each) run the same fast kernel as the unsharded 3 MiB fit
    -- weights and losses agree to 1e-12 (only the image norm's summation
    order differs)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_path_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    import paper_1608_01398_b200 as gi

    y = out[0][1]
    full = gi.PackedGenotypeMatrix.synthetic(1000, 12000, 31)
    # the unsharded path on the same (lookup-table) kernel -- not in a
    # tensor-core lock-step group, which sharded fits never use
    monkeypatch.setenv("GI_BATCH", "0")
    want = gi.fit_path(gi.StandardizedView(full, gi.CovariateBlock.build(None, n=1000)), y,
                       [3, 8, 12])
    for _, _, fits in out:
        for (support, weights, trace, iters), w in zip(fits, want):
            np.testing.assert_array_equal(support, w.model.support)
            assert iters == w.iterations
            np.testing.assert_allclose(weights, w.model.weights, rtol=1e-12, atol=0)
            np.testing.assert_allclose(trace, w.loss_trace, rtol=1e-12, atol=0)


def _nccl_multi_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_1608_01398_b200 as gi
        from paper_1608_01398_b200.dist import ShardedGenotypes, TorchComm
        from paper_1608_01398_b200.simulate import SimulationSpec, simulate_phenotype

        comm = TorchComm()
        geno = ShardedGenotypes.synthetic(N, P, SEED, comm, device=rank, missing_rate=0.01)
        view = gi.StandardizedView(geno, gi.CovariateBlock.build(None, n=N))
        y, _ = simulate_phenotype(view, SimulationSpec(k_true=K, seed=5))
        res = gi.fit(view, y, gi.IhtConfig(k=K))
        q.put((rank, y, res.model.support, res.model.weights, res.loss_trace, res.iterations,
               geno.native_comm().kind))
    finally:
        dist.destroy_process_group()


def test_nccl_two_or_more_gpus_match_single_device_fit():
    """The production multi-GPU path: one process per GPU, NCCL communicator,
    in-place device all-reduces and all-gathers across ranks.  Needs >= 2
    GPUs (the round-end pool has one; skipped there, runs on any multi-GPU
    node)."""
    import torch

    world = min(torch.cuda.device_count(), 8)
    if world < 2:
        pytest.skip(f"needs >= 2 GPUs for cross-GPU NCCL ranks (found {world})")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_multi_worker, args=(r, world, port, q))
             for r in range(world)]
    for p_ in procs:
        p_.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    import paper_1608_01398_b200 as gi

    y = out[0][1]
    full = gi.PackedGenotypeMatrix.synthetic(N, P, SEED, missing_rate=0.01)
    want = gi.fit(gi.StandardizedView(full, gi.CovariateBlock.build(None, n=N)), y,
                  gi.IhtConfig(k=K))
    for rank, _, support, weights, trace, iters, kind in out:
        assert kind == "nccl"
        np.testing.assert_array_equal(support, want.model.support)
        assert iters == want.iterations
        np.testing.assert_allclose(weights, want.model.weights, rtol=1e-9)
        np.testing.assert_allclose(trace, want.loss_trace, rtol=1e-9)
