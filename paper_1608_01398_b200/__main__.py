"""``python -m paper_1608_01398_b200 bench ...`` -- the reference's ``genoiht
bench`` (cli.py:285-353) with a ``gpu`` mode.

Times the model-size path (one cold fit per budget, IhtConfig(k, max_iter,
tol)) on the device and writes ``<out>.bench.tsv`` (mode, repetitions,
mean_seconds, sd_seconds, rel_to_dense) and ``<out>.bench_models.tsv`` (mode,
k, support) with the reference's ``# genoiht=... command=... config=...
seed=...`` first line.  ``--synthetic n,p`` generates genotypes on the device
(law of random_packed_matrix, counter-based stream); ``--bed/--n/--p`` reads a
BED file.  Modes: ``gpu`` (the path's fits concurrently, in a lock-step group
when large enough), ``gpu+seq`` (one fit at a time, as the reference's loop),
``dense`` (the reference's own uncompressed DenseDesign on the host, from
baseline/_ref: the denominator of rel_to_dense, as in the reference).  The
rest of the reference CLI (fit/cv/simulate, BIM/FAM text) is out of scope for
this build.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

from . import (CovariateBlock, IhtConfig, PackedGenotypeMatrix, StandardizedView, __version__,
               fit, fit_path, read_bed)
from .simulate import SimulationSpec, simulate_phenotype


def _path_spec(text: str) -> np.ndarray:
    if ":" in text:
        start, stop, step = (int(tok) for tok in text.split(":"))
        if step < 1 or stop < start:
            raise SystemExit(f"bad path specification {text!r}; use a:b:step or k1,k2,...")
        return np.arange(start, stop + 1, step, dtype=np.int64)
    path = np.unique(np.array([int(tok) for tok in text.split(",") if tok], dtype=np.int64))
    if path.size == 0 or path.min() < 1:
        raise SystemExit("path budgets must be integers >= 1")
    return path


def _config_hash(args) -> str:
    skip = {"out", "threads", "func", "command"}
    blob = json.dumps({k: v for k, v in sorted(vars(args).items()) if k not in skip},
                      default=str, sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()[:12]


def _fmt(v) -> str:
    if isinstance(v, float):
        return "nan" if v != v else f"{v:.10g}"
    return str(v)


def _table(path: Path, meta: str, header, rows) -> None:
    with open(path, "w") as fh:
        fh.write(meta + "\n" + "\t".join(header) + "\n")
        for row in rows:
            fh.write("\t".join(_fmt(c) for c in row) + "\n")


def cmd_bench(args) -> int:
    if args.synthetic:
        n, p = (int(t) for t in args.synthetic.split(","))
        geno = PackedGenotypeMatrix.synthetic(n, p, args.seed, device=args.device)
    else:
        geno = read_bed(args.bed, args.n, args.p, device=args.device)
    view = StandardizedView(geno, CovariateBlock.build(None, n=geno.n))
    y, _ = simulate_phenotype(view, SimulationSpec(k_true=args.bench_k_true, seed=args.seed))
    path = _path_spec(args.path)
    path = path[path <= min(view.p, view.n - view.c - 1)]
    if path.size == 0:
        raise SystemExit("no path budgets usable")
    modes = [m.strip() for m in args.mode.split(",") if m.strip()]
    known = {"gpu", "gpu+seq", "dense"}
    if set(modes) - known:
        raise SystemExit(f"unknown bench mode(s) {sorted(set(modes) - known)}; "
                         f"choose from {sorted(known)}")
    cfg = IhtConfig(k=int(path.max()), max_iter=args.max_iter, tol=args.tol)
    fit(view, y, cfg)  # warm the device path
    timings, model_rows = {}, []
    for mode in modes:
        durations = []
        run_dense = _dense_runner(args, geno, view, y, path) if mode == "dense" else None
        for rep in range(args.repetitions):
            start = time.perf_counter()
            if mode == "gpu":
                results = fit_path(view, y, path, cfg)
            elif mode == "dense":
                results = run_dense()
            else:  # one fit at a time, as the reference's loop
                results = [fit(view, y, IhtConfig(k=int(k), max_iter=args.max_iter,
                                                  tol=args.tol)) for k in path]
            durations.append(time.perf_counter() - start)
            if rep == 0:
                for k, res in zip(path, results):
                    model_rows.append((mode, int(k),
                                       ",".join(str(int(j)) for j in res.model.support)))
        timings[mode] = (float(np.mean(durations)),
                         float(np.std(durations, ddof=1)) if len(durations) > 1 else 0.0)
    meta = (f"# genoiht={__version__} command=bench config={_config_hash(args)} "
            f"seed={args.seed}")
    # rel_to_dense as the reference writes it (cli.py:337-343): a mode's mean
    # over the dense mode's, NaN when dense was not run
    dense_mean = timings["dense"][0] if "dense" in timings else float("nan")
    rows = [(m, args.repetitions, timings[m][0], timings[m][1], timings[m][0] / dense_mean)
            for m in modes]
    _table(Path(args.out + ".bench.tsv"), meta,
           ["mode", "repetitions", "mean_seconds", "sd_seconds", "rel_to_dense"], rows)
    _table(Path(args.out + ".bench_models.tsv"), meta, ["mode", "k", "support"], model_rows)
    for m in modes:
        print(f"bench {m}: {timings[m][0]:.3f}s mean, {timings[m][1]:.3f}s sd over "
              f"{args.repetitions} reps")
    return 0


def _dense_runner(args, geno, view, y, path):
    """The reference's ``dense`` bench mode (cli.py:303-315): genoiht's own
    DenseDesign (the uncompressed float design, numpy BLAS on the host) built
    from the same bytes, fitted by genoiht's loop -- the paper's uncompressed
    baseline (Table 1), so rel_to_dense is the device path's speed-up
    over it.  Needs the reference package (baseline/_ref)."""
    import os

    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "genoiht")):
        raise SystemExit("dense mode needs the reference package in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/genoiht_numba_cache")
    sys.path.insert(0, ref_dir)
    import genoiht

    estimate = 8 * view.n * view.p
    if estimate > int(args.mem_cap_gb * 2 ** 30):
        raise SystemExit(f"dense mode refused: {estimate / 2 ** 30:.2f} GiB uncompressed "
                         f"exceeds the {args.mem_cap_gb} GiB cap")
    host = genoiht.PackedGenotypeMatrix.from_bed_buffer(np.array(geno.data), geno.n)
    design = genoiht.DenseDesign.from_packed(host, dtype=np.float64)
    dview = genoiht.StandardizedView(design, genoiht.CovariateBlock.build(None, n=geno.n))
    genoiht.set_worker_threads(args.threads)

    def run():
        return [genoiht.fit(dview, y, genoiht.IhtConfig(k=int(k), max_iter=args.max_iter,
                                                        tol=args.tol)) for k in path]
    return run


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1608_01398_b200")
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="time the model-size path on the GPU")
    src = b.add_mutually_exclusive_group(required=True)
    src.add_argument("--synthetic", help="n,p of device-generated genotypes")
    src.add_argument("--bed", help="PLINK .bed file (with --n, --p)")
    b.add_argument("--n", type=int)
    b.add_argument("--p", type=int)
    b.add_argument("--path", default="5:100:5")
    b.add_argument("--mode", default="gpu")
    b.add_argument("--repetitions", type=int, default=3)
    b.add_argument("--bench-k-true", type=int, default=10)
    b.add_argument("--max-iter", type=int, default=200)
    b.add_argument("--tol", type=float, default=1e-4)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--device", type=int, default=0)
    b.add_argument("--threads", type=int, default=8, help="host threads of the dense mode")
    b.add_argument("--mem-cap-gb", type=float, default=32.0,
                   help="refuse the dense mode beyond this many GiB of uncompressed design")
    b.add_argument("--out", required=True)
    b.set_defaults(func=cmd_bench)
    args = ap.parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
