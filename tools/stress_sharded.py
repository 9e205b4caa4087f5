"""Randomised parity stress of the SHARDED native loop (gi_fit_sharded): two
processes share one GPU, each owning a contiguous SNP block (host-staged gloo
collectives, so no kernel waits on the other rank), over random problems --
ragged shapes, missing data, covariates, warm starts, duplicated columns
across the shard boundary, unequal and empty shards.  Rank 0 compares each
sharded fit with the oracle (support, iterations and reason exact; beta,
b_cov and loss within 1e-6 of the vector).

    python tools/stress_sharded.py [cases] [seed0]
"""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

RTOL = 1e-6


def problem(seed):
    import oracle

    rng = np.random.default_rng(seed)
    n = int(rng.integers(40, 2000))
    p = int(rng.integers(8, 5000))
    miss = float(rng.choice([0.0, 0.0, 0.02, 0.1]))
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    if rng.random() < 0.3:  # duplicates, some straddling the shard boundary
        dup = rng.choice(p, min(6, p // 2), replace=False)
        codes[:, (dup + p // 2) % p] = codes[:, dup]
    covar = rng.standard_normal((n, int(rng.choice([0, 1, 3])))) if rng.random() < 0.5 else None
    if covar is not None and covar.shape[1] == 0:
        covar = None
    k = int(rng.integers(1, 20))
    support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 7))), replace=False))
    weights = rng.standard_normal(support.size)
    noise = float(rng.choice([0.01, 0.3, 1.0]))
    eps = rng.normal(0, noise, n)
    split = [None, 0, p][int(rng.integers(0, 3))] if rng.random() < 0.15 else None
    warm = None
    if rng.random() < 0.2:
        widx = np.sort(rng.choice(p, min(p, k, 3), replace=False))
        warm = (widx, rng.standard_normal(widx.size))
    return n, p, codes, covar, k, support, weights, eps, split, warm


def worker(rank, world, port, seeds, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import oracle
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200.dist import ShardedGenotypes, TorchComm, shard_range

    comm = TorchComm()
    oracle.set_threads(max(1, (os.cpu_count() or 2) // 2))
    for seed in seeds:
        n, p, codes, covar, k, support, weights, eps, split, warm = problem(seed)
        j0, j1 = shard_range(p, world, rank)
        if split is not None:  # an empty shard on one side
            j0, j1 = (0, split) if rank == 0 else (split, p)
        local = gi.PackedGenotypeMatrix.from_codes(codes[:, j0:j1])
        geno = ShardedGenotypes(local, j0, p, comm)
        block = gi.CovariateBlock.build(covar, n=n)
        view = gi.StandardizedView(geno, block)
        ref_geno = oracle.OraclePacked.from_codes(codes)
        y = ref_geno.ax_columns(support, weights) + eps
        wm = None
        if warm is not None:
            wm = gi.SparseModel.from_parts(warm[0], warm[1], np.zeros(block.c), k=k, p=p)
        try:
            got = gi.fit(view, y, gi.IhtConfig(k=k), warm=wm)
            err = None
        except Exception as exc:  # noqa: BLE001
            got, err = None, f"{type(exc).__name__}: {exc}"
            print(f"rank {rank} seed {seed}: {err}", flush=True)
        if rank == 0:
            try:
                want = oracle.fit(oracle.OracleView(ref_geno, block.values), y, k,
                                  warm=None if warm is None else (warm[0], warm[1],
                                                                  np.zeros(block.c)))
                werr = None
            except Exception as exc:  # noqa: BLE001
                want, werr = None, type(exc).__name__
            desc = f"seed={seed} n={n} p={p} k={k} c={block.c} shards=[{j0},{j1}) " \
                   f"warm={warm is not None}"
            if err or werr:
                q.put((seed, err is not None and werr is not None,
                       desc + f" errors: device {err} oracle {werr}"))
                continue
            problems = []
            if not np.array_equal(got.model.support, want.support):
                problems.append("support")
            if got.iterations != want.iterations or got.reason != want.reason:
                problems.append(f"iterations {got.iterations}/{want.iterations}")
            for name, a, b in (("weights", got.model.weights, want.weights),
                               ("covar", got.model.covar, want.covar),
                               ("loss", got.loss_trace, want.loss_trace)):
                a, b = np.asarray(a, float), np.asarray(b, float)
                if b.size and a.shape == b.shape and \
                        np.max(np.abs(a - b)) > RTOL * np.max(np.abs(b)) + 1e-12:
                    problems.append(f"{name} {np.max(np.abs(a - b)) / np.max(np.abs(b)):.1e}")
            q.put((seed, not problems, desc + (" " + ", ".join(problems) if problems else "")))
    dist.destroy_process_group()


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 110000
    seeds = list(range(seed0, seed0 + cases))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, 2, port, seeds, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    bad = 0
    for _ in seeds:
        seed, ok, desc = q.get(timeout=300)
        if not ok:
            bad += 1
            print("MISMATCH", desc, flush=True)
    for p_ in procs:
        p_.join(timeout=120)
    print(f"{cases - bad}/{cases} sharded cases match the oracle", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
