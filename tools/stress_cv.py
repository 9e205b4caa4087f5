"""Randomised parity stress of cross-validation: cv_iht on the device (compact
or masked folds, concurrent fits) vs the oracle's cv (the reference's per-fold
re-pack and loop) on random problems -- q = 3-5 folds, paths up to k = 10,
train / global standardisation, warm / cold starts, covariates, missing data.
k_best and the final support must be equal; the per-fold MSE grid within
1e-5 and the final model within 1e-6 of the vector.

    python tools/stress_cv.py [cases] [seed0]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_1608_01398_b200 as gi  # noqa: E402


def case(seed):
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
    desc = f"seed={seed} n={n} p={p} q={q} path=1..{path.max()} {std_mode} warm={warm} " \
           f"c={block.c} miss={miss}"
    try:
        want = oracle.cv(oracle.OracleView(ref_p, block.values), y, q, path, seed,
                         std_mode=std_mode, warm_start=warm, labels=plan.fold_labels)
        werr = None
    except Exception as exc:  # noqa: BLE001
        want, werr = None, type(exc).__name__
    try:
        got = gi.cv_iht(view, y, plan, gi.IhtConfig(k=int(path.max())), std_mode=std_mode,
                        warm_start=warm)
        gerr = None
    except Exception as exc:  # noqa: BLE001
        got, gerr = None, type(exc).__name__
    if werr or gerr:
        return (werr is not None) == (gerr is not None), desc + f" errors {werr}/{gerr}"
    problems = []
    if got.k_best != want.k_best:
        problems.append(f"k_best {got.k_best} vs {want.k_best}")
    if np.max(np.abs(got.mse - want.mse)) > 1e-5 * np.max(np.abs(want.mse)):
        problems.append("mse")
    f_sup, f_w, f_cov = want.final  # oracle.refit -> (support, weights, covar)
    if not np.array_equal(got.final_model.support, f_sup):
        problems.append("final support")
    else:
        for name, a, b in (("weights", got.final_model.weights, f_w),
                           ("covar", got.final_model.covar, f_cov)):
            if b.size and np.max(np.abs(a - b)) > 1e-6 * np.max(np.abs(b)) + 1e-12:
                problems.append(name)
    return not problems, desc + (" " + ", ".join(problems) if problems else "")


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 130000
    oracle.set_threads(os.cpu_count() or 1)
    bad = 0
    for s in range(seed0, seed0 + cases):
        ok, desc = case(s)
        if not ok:
            bad += 1
            print("MISMATCH", desc, flush=True)
    print(f"{cases - bad}/{cases} CV cases match the oracle", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
