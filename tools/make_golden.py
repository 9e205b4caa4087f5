"""Generate golden vectors from the REFERENCE implementation (genoiht 0.1.0).

Runs only in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/make_golden.py

Writes tests/golden/*.npz.  Inputs are regenerated from seeds by the tests
(oracle.random_codes replays the reference's numpy draws); every fixture stores
a SHA-256 of the packed bytes so a drifting generator is caught, plus the
reference outputs: stats, X^T r, X_S w, decompressed columns, fit results and
cross-validation reports.  The GPU box never reads /root/reference; it only
reads these committed fixtures.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import genoiht  # noqa: E402
from genoiht import (CovariateBlock, CvPlan, IhtConfig, PackedGenotypeMatrix,  # noqa: E402
                     SimulationSpec, StandardizedView, cv_iht, fit, simulate_phenotype)
from genoiht.simulate import random_packed_matrix  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def sha(data: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(data).tobytes()).hexdigest()


def random_codes_ref(n, p, seed, missing_rate):
    # identical draws to simulate.random_packed_matrix, returning codes
    m = random_packed_matrix(n, p, seed=seed, missing_rate=missing_rate)
    return m.to_codes()


def kernel_cases():
    cases = []
    rng = np.random.default_rng(424242)
    shapes = [(5, 2, 0.0), (7, 3, 0.2), (13, 9, 0.1), (20, 50, 0.15), (16, 12, 0.1),
              (97, 300, 0.05), (403, 517, 0.1), (1000, 257, 0.02), (1, 4, 0.0), (6, 1, 1.0)]
    for ci, (n, p, miss) in enumerate(shapes):
        seed = 9000 + ci
        codes = random_codes_ref(n, p, seed, miss) if miss < 1.0 else np.full((n, p), 1, np.uint8)
        m = PackedGenotypeMatrix.from_codes(codes)
        r = rng.standard_normal(n)
        kk = max(1, min(p, 1 + ci % 7))
        support = np.sort(rng.choice(p, kk, replace=False)).astype(np.int64)
        weights = rng.standard_normal(kk)
        dense_idx = np.arange(p, dtype=np.int64)
        dense_w = rng.standard_normal(p)
        cases.append(dict(
            name=f"kernel{ci}", n=n, p=p, seed=seed, missing=miss,
            all_missing=(miss >= 1.0), data_sha=sha(m.data), u=m.u, v=m.v, r=r,
            aty=m.aty_genetic(r) if p else np.zeros(0), support=support, weights=weights,
            ax=m.ax_columns(support, weights), dense_w=dense_w,
            ax_dense=m.ax_columns(dense_idx, dense_w),
            decompress=m.decompress(support)))
    return cases


def fit_cases():
    cases = []
    # BASELINE config 1: n=1000, p=10000, k=10, reference generator seeds
    specs = [
        dict(name="c1", n=1000, p=10000, seed=1608, missing=0.0, k_true=10, pheno_seed=1398,
             ks=[10], intercept=True),
        dict(name="small_miss", n=200, p=500, seed=77, missing=0.05, k_true=5, pheno_seed=78,
             ks=[1, 3, 5, 8, 12], intercept=True),
        dict(name="odd_n", n=333, p=1001, seed=91, missing=0.02, k_true=7, pheno_seed=92,
             ks=[4, 7, 9], intercept=True),
        dict(name="no_cov", n=150, p=400, seed=55, missing=0.0, k_true=4, pheno_seed=56,
             ks=[2, 4, 6], intercept=False),
        dict(name="c2_slice", n=5000, p=20000, seed=1608, missing=0.0, k_true=20,
             pheno_seed=1398, ks=[10, 20, 30], intercept=True),
    ]
    for sp in specs:
        codes = random_codes_ref(sp["n"], sp["p"], sp["seed"], sp["missing"])
        m = PackedGenotypeMatrix.from_codes(codes)
        cov = CovariateBlock.build(None, n=sp["n"]) if sp["intercept"] else None
        view = StandardizedView(m, cov)
        y, truth = simulate_phenotype(view, SimulationSpec(k_true=sp["k_true"],
                                                           seed=sp["pheno_seed"]))
        for k in sp["ks"]:
            res = fit(view, y, IhtConfig(k=k))
            cases.append(dict(
                name=f"{sp['name']}_k{k}", n=sp["n"], p=sp["p"], seed=sp["seed"],
                missing=sp["missing"], intercept=sp["intercept"], k=k, data_sha=sha(m.data),
                y=y, truth=truth.support, support=res.model.support, weights=res.model.weights,
                covar=res.model.covar, loss_trace=res.loss_trace, iterations=res.iterations,
                converged=res.converged, reason=res.reason))
    # k = 0 and a zero response (test_iht.py:179-184, :352-356 analogues on packed data)
    codes = random_codes_ref(40, 30, 5, 0.1)
    m = PackedGenotypeMatrix.from_codes(codes)
    for name, cov, y, k in [("zero_resp", CovariateBlock.build(None, n=40), np.zeros(40), 3),
                            ("k0_nocov", None, np.random.default_rng(6).standard_normal(40), 0),
                            ("k0_cov", CovariateBlock.build(None, n=40),
                             np.random.default_rng(7).standard_normal(40), 0)]:
        res = fit(StandardizedView(m, cov), y, IhtConfig(k=k))
        cases.append(dict(
            name=name, n=40, p=30, seed=5, missing=0.1, intercept=cov is not None, k=k,
            data_sha=sha(m.data), y=y, truth=np.zeros(0, np.int64),
            support=res.model.support, weights=res.model.weights, covar=res.model.covar,
            loss_trace=res.loss_trace, iterations=res.iterations, converged=res.converged,
            reason=res.reason))
    return cases


def cv_cases():
    cases = []
    specs = [
        dict(name="cv_planted", n=150, p=80, seed=42, q=5, path=np.arange(1, 9), fold_seed=3,
             std_mode="train", warm=False, support=[10, 40, 71], w=[1.0, -1.2, 0.9], noise=0.0),
        dict(name="cv_global", n=100, p=40, seed=31, q=4, path=np.arange(1, 6), fold_seed=7,
             std_mode="global", warm=False, support=[3, 30], w=[1.0, -1.0], noise=0.0),
        dict(name="cv_warm", n=300, p=60, seed=21, q=5, path=np.arange(1, 9), fold_seed=6,
             std_mode="train", warm=True, support=[5, 25, 45], w=[1.0, -1.0, 0.8], noise=0.05),
        dict(name="cv_mid", n=2000, p=3000, seed=2016, q=5, path=np.arange(1, 11), fold_seed=2016,
             std_mode="train", warm=False, support=[7, 300, 1500, 2999], w=[0.3, -0.2, 0.25, 0.1],
             noise=0.3),
    ]
    from genoiht.geno_matrix import ax_parts
    for sp in specs:
        codes = random_codes_ref(sp["n"], sp["p"], sp["seed"], 0.0)
        m = PackedGenotypeMatrix.from_codes(codes)
        view = StandardizedView(m, CovariateBlock.build(None, n=sp["n"]))
        y = ax_parts(view, np.array(sp["support"]), np.array(sp["w"]))
        if sp["noise"] > 0:
            y = y + np.random.default_rng(sp["seed"] + 1).normal(0.0, sp["noise"], sp["n"])
        plan = CvPlan.build(sp["n"], sp["q"], sp["path"], seed=sp["fold_seed"])
        rep = cv_iht(view, y, plan, IhtConfig(k=int(sp["path"].max())), std_mode=sp["std_mode"],
                     warm_start=sp["warm"])
        cases.append(dict(
            name=sp["name"], n=sp["n"], p=sp["p"], seed=sp["seed"], q=sp["q"], path=sp["path"],
            fold_seed=sp["fold_seed"], std_mode=sp["std_mode"], warm=sp["warm"],
            data_sha=sha(m.data), y=y, labels=plan.fold_labels, mse=rep.mse,
            mean_mse=rep.mean_mse, k_best=rep.k_best, final_support=rep.final_model.support,
            final_weights=rep.final_model.weights, final_covar=rep.final_model.covar))
    return cases


def _synth_matrix(n, p, seed, missing):
    """The device generator's bytes (its CPU twin in oracle/), as a reference
    matrix: the GPU tests rebuild the same matrix with
    PackedGenotypeMatrix.synthetic(n, p, seed, missing_rate=missing)."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
    import oracle
    data = oracle.synth_bed(seed, n, 0, p, missing=missing)
    return PackedGenotypeMatrix.from_bed_buffer(data, n)


def large_cases():
    """Fits and CV runs big enough for the native loop's FAST X^T r kernel
    (> 2 MiB of tiles and n > 8 (k + c + 1): csrc/fit.cu NativeFit), with and
    without missing genotypes (2-bit tiles with the missing-sum lookups, or
    the base-3 copy), covariates, warm starts and both CV standardisations."""
    cases = []
    fit_specs = [
        dict(name="fit_miss3", n=4000, p=20000, seed=4242, missing=0.03, k_true=12,
             pheno_seed=11, ks=[6, 12, 25], ncov=0),
        dict(name="fit_miss2_cov", n=4100, p=16000, seed=4343, missing=0.02, k_true=10,
             pheno_seed=12, ks=[10, 18], ncov=2),
        dict(name="fit_base3_cov", n=3333, p=24000, seed=4444, missing=0.0, k_true=15,
             pheno_seed=13, ks=[15], ncov=1),
    ]
    for sp in fit_specs:
        m = _synth_matrix(sp["n"], sp["p"], sp["seed"], sp["missing"])
        raw = None
        if sp["ncov"]:
            raw = np.random.default_rng(sp["seed"] + 7).standard_normal((sp["n"], sp["ncov"]))
        view = StandardizedView(m, CovariateBlock.build(raw, n=sp["n"]))
        y, truth = simulate_phenotype(view, SimulationSpec(k_true=sp["k_true"],
                                                           seed=sp["pheno_seed"]))
        for k in sp["ks"]:
            res = fit(view, y, IhtConfig(k=k))
            cases.append(dict(
                kind="fit", name=f"{sp['name']}_k{k}", n=sp["n"], p=sp["p"], seed=sp["seed"],
                missing=sp["missing"], k=k, covar_raw=raw if raw is not None else np.zeros(0),
                data_sha=sha(m.data), y=y, truth=truth.support, support=res.model.support,
                weights=res.model.weights, covar=res.model.covar, loss_trace=res.loss_trace,
                iterations=res.iterations, reason=res.reason))
    cv_specs = [
        dict(name="cvL_train_cold", n=3000, p=12000, seed=5151, missing=0.0, q=5,
             path=np.arange(1, 9), fold_seed=2016, std_mode="train", warm=False),
        dict(name="cvL_global_cold", n=3000, p=12000, seed=5151, missing=0.0, q=5,
             path=np.arange(1, 9), fold_seed=2016, std_mode="global", warm=False),
        dict(name="cvL_train_warm_miss", n=2600, p=14000, seed=5252, missing=0.02, q=4,
             path=np.arange(2, 12, 2), fold_seed=77, std_mode="train", warm=True),
        dict(name="cvL_global_warm_miss", n=2600, p=14000, seed=5252, missing=0.02, q=4,
             path=np.arange(2, 12, 2), fold_seed=77, std_mode="global", warm=True),
        # cold starts with missing genotypes: the lock-step group's tensor-core
        # sweeps with the missing-flag MMAs, and the base-3 copy + missing list
        dict(name="cvL_train_cold_miss", n=2600, p=14000, seed=5353, missing=0.02, q=4,
             path=np.arange(1, 9), fold_seed=91, std_mode="train", warm=False),
        dict(name="cvL_global_cold_miss", n=2600, p=14000, seed=5353, missing=0.02, q=4,
             path=np.arange(1, 9), fold_seed=91, std_mode="global", warm=False),
    ]
    for sp in cv_specs:
        m = _synth_matrix(sp["n"], sp["p"], sp["seed"], sp["missing"])
        view = StandardizedView(m, CovariateBlock.build(None, n=sp["n"]))
        y, truth = simulate_phenotype(view, SimulationSpec(k_true=6, seed=sp["seed"] + 1))
        plan = CvPlan.build(sp["n"], sp["q"], sp["path"], seed=sp["fold_seed"])
        rep = cv_iht(view, y, plan, IhtConfig(k=int(sp["path"].max())), std_mode=sp["std_mode"],
                     warm_start=sp["warm"])
        cases.append(dict(
            kind="cv", name=sp["name"], n=sp["n"], p=sp["p"], seed=sp["seed"],
            missing=sp["missing"], q=sp["q"], path=sp["path"], fold_seed=sp["fold_seed"],
            std_mode=sp["std_mode"], warm=sp["warm"], data_sha=sha(m.data), y=y,
            labels=plan.fold_labels, mse=rep.mse, mean_mse=rep.mean_mse, k_best=rep.k_best,
            final_support=rep.final_model.support, final_weights=rep.final_model.weights,
            final_covar=rep.final_model.covar))
    return cases


def main():
    os.makedirs(OUT, exist_ok=True)
    groups = [("kernels", kernel_cases), ("fits", fit_cases), ("cv", cv_cases),
              ("large", large_cases)]
    only = sys.argv[1:]
    for group, fn in groups:
        if only and group not in only:
            continue
        cases = fn()
        payload = {}
        for c in cases:
            for key, val in c.items():
                payload[f"{c['name']}__{key}"] = np.asarray(val)
        payload["__cases"] = np.array([c["name"] for c in cases])
        payload["__reference_version"] = np.array(genoiht.__version__)
        np.savez_compressed(os.path.join(OUT, f"{group}.npz"), **payload)
        print(group, len(cases), "cases")


if __name__ == "__main__":
    main()
