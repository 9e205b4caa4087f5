"""Randomised parity stress: native device fits vs the oracle (reference
algorithm) over many random problems -- shapes with ragged tiles/groups,
missing rates, covariates, budgets from 1 to above the support, warm starts,
masked CV folds and duplicated columns (exact ties in the top-k).  Prints one
line per mismatch and a summary; exit code 1 on any mismatch.

    python tools/stress_parity.py [cases] [seed0]
    GI_STRESS_LARGE=1 python tools/stress_parity.py ...   # larger shapes (fast kernel)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402
from paper_1608_01398_b200.model_select import FoldGenotypes  # noqa: E402

RTOL = 1e-6


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    if a.size == 0 and b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


LARGE = os.environ.get("GI_STRESS_LARGE") == "1"  # n up to 20k, p up to 120k: fast-kernel plans


def build_large(seed):
    """Larger problems from the device generator and its CPU twin (same bytes,
    no dense code matrix on the host): the fast kernel's multi-item and
    tile-sliced work plans, masked folds, covariates, warm starts."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2000, 20000))
    p = int(rng.integers(5000, 120000))
    miss = float(rng.choice([0.0, 0.0, 0.02]))
    m = gi.PackedGenotypeMatrix.synthetic(n, p, seed, missing_rate=miss)
    ref_p = oracle.OraclePacked.from_bed(oracle.synth_bed(seed, n, 0, p, missing=miss), n)
    c_extra = int(rng.choice([0, 0, 2]))
    covar = rng.standard_normal((n, c_extra)) if c_extra else None
    block = gi.CovariateBlock.build(covar, n=n)
    k = int(rng.integers(1, 40))
    support = np.sort(rng.choice(p, int(rng.integers(1, 12)), replace=False))
    y = ref_p.ax_columns(support, rng.standard_normal(support.size)) \
        + rng.normal(0, float(rng.choice([0.05, 0.5])), n)
    warm = None
    if rng.random() < 0.2:
        widx = np.sort(rng.choice(p, min(k, 3), replace=False))
        warm = (widx, rng.standard_normal(widx.size), np.zeros(block.c))
    keep = np.flatnonzero(rng.random(n) < 0.8) if rng.random() < 0.25 else None
    if keep is not None:
        u, v = m.masked_stats(np.isin(np.arange(n), keep).astype(np.uint8))
        ref_view = oracle.OracleView(ref_p.subset_rows(keep), block.values[keep])
        view = gi.StandardizedView(FoldGenotypes(m.with_stats(u, v), keep),
                                   block.subset_rows(keep))
        y_fit = y[keep]
    else:
        ref_view = oracle.OracleView(ref_p, block.values)
        view = gi.StandardizedView(m, block)
        y_fit = y
    warm_model = None if warm is None else \
        gi.SparseModel.from_parts(warm[0], warm[1], warm[2], k=k, p=p)
    desc = f"seed={seed} n={n} p={p} k={k} miss={miss} c={block.c} " \
           f"masked={keep is not None} warm={warm is not None} (large)"
    return view, ref_view, y_fit, k, warm, warm_model, desc


def build(seed):
    """The random problem of `seed`: device view, oracle view, response, budget, warm start."""
    if LARGE:
        return build_large(seed)
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 2500))
    p = int(rng.integers(5, 6000))
    miss = float(rng.choice([0.0, 0.0, 0.01, 0.05, 0.2]))
    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    if rng.random() < 0.3 and p > 10:  # duplicated columns: exact ties
        dup = rng.choice(p, min(5, p // 2), replace=False)
        codes[:, (dup + 1) % p] = codes[:, dup]
    c_extra = int(rng.choice([0, 0, 1, 3]))
    covar = rng.standard_normal((n, c_extra)) if c_extra else None
    intercept = rng.random() < 0.8
    k = int(rng.integers(1, 25))
    keep = None
    if rng.random() < 0.25:
        keep = np.flatnonzero(rng.random(n) < 0.8)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    block = gi.CovariateBlock.build(covar, n=n, add_intercept=intercept) \
        if (covar is not None or intercept) else None
    ref_p = oracle.OraclePacked.from_codes(codes)
    support = np.sort(rng.choice(p, min(p, int(rng.integers(1, 8))), replace=False))
    y = ref_p.ax_columns(support, rng.standard_normal(support.size)) \
        + rng.normal(0, float(rng.choice([0.01, 0.3, 1.0])), n)
    warm = None
    if rng.random() < 0.2:
        widx = np.sort(rng.choice(p, min(p, k, 3), replace=False))
        warm = (widx, rng.standard_normal(widx.size), np.zeros(0 if block is None else block.c))
    if keep is not None:
        u, v = m.masked_stats(np.isin(np.arange(n), keep).astype(np.uint8))
        sub_codes = codes[keep]
        ref_view = oracle.OracleView(oracle.OraclePacked.from_codes(sub_codes),
                                     None if block is None else block.values[keep])
        fold = FoldGenotypes(m.with_stats(u, v), keep)
        view = gi.StandardizedView(fold, None if block is None else block.subset_rows(keep))
        y_fit = y[keep]
    else:
        ref_view = oracle.OracleView(ref_p, None if block is None else block.values)
        view = gi.StandardizedView(m, block)
        y_fit = y
    warm_model = None
    if warm is not None:
        warm_model = gi.SparseModel.from_parts(warm[0], warm[1], warm[2], k=k, p=p)
    desc = f"seed={seed} n={n} p={p} k={k} miss={miss} c={0 if block is None else block.c} " \
           f"masked={keep is not None} warm={warm is not None}"
    return view, ref_view, y_fit, k, warm, warm_model, desc


def case(seed):
    view, ref_view, y_fit, k, warm, warm_model, desc = build(seed)
    cfg = gi.IhtConfig(k=k)
    try:
        want = oracle.fit(ref_view, y_fit, k, warm=warm)
        want_err = None
    except Exception as exc:  # the reference raises too: the device must match
        want, want_err = None, type(exc)
    try:
        got = gi.fit(view, y_fit, cfg, warm=warm_model)
        got_err = None
    except Exception as exc:
        got, got_err = None, type(exc)
    if want_err or got_err:
        ok = want_err is not None and got_err is not None
        return ok, desc + f" errors: oracle {want_err} device {got_err}"
    problems, notes = [], []
    if not np.array_equal(got.model.support, want.support):
        problems.append("support")
    if got.iterations != want.iterations:
        problems.append(f"iterations {got.iterations} vs {want.iterations}")
    if got.reason != want.reason:
        problems.append(f"reason {got.reason} vs {want.reason}")
    if not problems:
        for name, a, b in (("weights", got.model.weights, want.weights),
                           ("covar", got.model.covar, want.covar),
                           ("loss", got.loss_trace, want.loss_trace)):
            # 1e-6 relative to the vector (max-norm), as in tests/test_gpu_fit.py
            a, b = np.asarray(a, float), np.asarray(b, float)
            scale = float(np.max(np.abs(b))) if b.size else 0.0
            err = float(np.max(np.abs(a - b))) if b.size else 0.0
            if err > RTOL * scale + 1e-12:
                problems.append(f"{name} {err / max(scale, 1e-300):.2e} of max")
            elif rel(a, b) > RTOL:
                notes.append(f"{name} elementwise {rel(a, b):.1e}")
    return not problems, desc + (" " + ", ".join(problems + notes) if problems or notes else "")


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
    oracle.set_threads(os.cpu_count() or 1)
    bad = 0
    for s in range(seed0, seed0 + cases):
        ok, desc = case(s)
        if not ok:
            bad += 1
            print("MISMATCH", desc, flush=True)
        elif "elementwise" in desc:
            print("note", desc, flush=True)
    print(f"{cases - bad}/{cases} cases match the oracle", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
