"""Parity of the native loop's FAST X^T r kernels against the reference.

The golden fits and CV runs in tests/golden/large.npz (tools/make_golden.py,
produced by genoiht 0.1.0 itself) are big enough that the native loop runs
the lookup-table X^T r kernel, not the exact fp64 one (more than 2 MiB of
tiles and n > 8 (k + c + 1); csrc/fit.cu NativeFit): over the base-3 copy,
with the missing-genotype list when genotypes are missing (2-3%), and for
those also over the 2-bit tiles with the missing-sum lookups.  The matrices are rebuilt on the device by the
generator whose CPU twin made the reference's bytes (checked by SHA-256).

Bar (north star): support, iteration count and reason identical; beta, b_cov
and the loss trace within 1e-6 relative (vector reading: see
test_gpu_fit.vec_atol); CV: k_best, the fold-mean MSE curve, the final
model.  CV runs both ways the device holds training folds: compact device
copies (GI_CV_COMPACT=1) and row masks over the resident matrix (=0).
"""
import numpy as np
import pytest

import golden_io

pytestmark = pytest.mark.gpu

RTOL = 1e-6
LARGE = golden_io.load("large")
FITS = sorted(k for k, v in LARGE.items() if v["kind"] == "fit")
CVS = sorted(k for k, v in LARGE.items() if v["kind"] == "cv")


def vec_atol(want):
    want = np.asarray(want, dtype=np.float64)
    return RTOL * float(np.max(np.abs(want))) if want.size else 0.0


def _matrix(case):
    import paper_1608_01398_b200 as gi

    m = gi.PackedGenotypeMatrix.synthetic(case["n"], case["p"], case["seed"],
                                          missing_rate=case["missing"])
    assert golden_io.sha(m.data) == case["data_sha"], "device generator drifted from the twin"
    return m


FIT_CASES = [(k, "1") for k in FITS] + [(k, "0") for k in FITS if LARGE[k]["missing"] > 0]


@pytest.mark.parametrize("name,misslist", FIT_CASES)
def test_large_fit_matches_reference(name, misslist, monkeypatch):
    """Missing genotypes: X^T r over the base-3 copy plus the missing list
    (GI_MISSLIST=1, the default) and over the 2-bit tiles (=0)."""
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200.iht import last_native_fit_info

    monkeypatch.setenv("GI_MISSLIST", misslist)
    case = LARGE[name]
    m = _matrix(case)
    raw = case["covar_raw"]
    block = gi.CovariateBlock.build(raw if raw.size else None, n=case["n"])
    res = gi.fit(gi.StandardizedView(m, block), case["y"], gi.IhtConfig(k=int(case["k"])))
    info = last_native_fit_info()
    want_kernel = "fast-base3" if case["missing"] == 0 else \
        ("fast-base3-misslist" if misslist == "1" else "fast-2bit")
    assert info["xtr_kernel"] == want_kernel, info
    np.testing.assert_array_equal(res.model.support, case["support"])
    assert res.iterations == case["iterations"] and res.reason == case["reason"]
    np.testing.assert_allclose(res.model.weights, case["weights"], rtol=RTOL,
                               atol=vec_atol(case["weights"]))
    np.testing.assert_allclose(res.model.covar, case["covar"], rtol=RTOL,
                               atol=vec_atol(case["covar"]) + 1e-12)
    np.testing.assert_allclose(res.loss_trace, case["loss_trace"], rtol=RTOL, atol=1e-12)


@pytest.mark.parametrize("compact", ["1", "0"], ids=["compact-folds", "masked-folds"])
@pytest.mark.parametrize("name", CVS)
def test_large_cv_matches_reference(name, compact, monkeypatch):
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200.iht import _xtr_exact

    monkeypatch.setenv("GI_CV_COMPACT", compact)
    case = LARGE[name]
    m = _matrix(case)
    # every fold fit is big enough for the fast kernel
    n_train = case["n"] - np.bincount(case["labels"]).max()
    assert not _xtr_exact(int(n_train), case["p"], int(case["path"].max()), 1)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=case["n"]))
    plan = gi.CvPlan.build(case["n"], case["q"], case["path"], seed=case["fold_seed"])
    np.testing.assert_array_equal(plan.fold_labels, case["labels"])
    rep = gi.cv_iht(view, case["y"], plan, gi.IhtConfig(k=int(case["path"].max())),
                    std_mode=case["std_mode"], warm_start=bool(case["warm"]))
    assert rep.k_best == case["k_best"]
    np.testing.assert_allclose(rep.mse, case["mse"], rtol=RTOL)
    np.testing.assert_allclose(rep.mean_mse, case["mean_mse"], rtol=RTOL)
    np.testing.assert_array_equal(rep.final_model.support, case["final_support"])
    np.testing.assert_allclose(rep.final_model.weights, case["final_weights"], rtol=RTOL,
                               atol=vec_atol(case["final_weights"]))
    np.testing.assert_allclose(rep.final_model.covar, case["final_covar"], rtol=RTOL,
                               atol=1e-12)


@pytest.mark.parametrize("name", [k for k in CVS if not LARGE[k]["warm"]])
def test_large_cv_lockstep_tensor_core_matches_reference(name, monkeypatch):
    """Cold-start CV with every (fold, budget) fit in one lock-step group: the
    fits' X^T r sweeps run together on the tensor cores (multi-RHS X^T R,
    csrc/batch.cu + xtr_mma.cu) -- same golden numbers."""
    import paper_1608_01398_b200 as gi

    monkeypatch.setenv("GI_BATCH", "1")
    case = LARGE[name]
    m = _matrix(case)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=case["n"]))
    plan = gi.CvPlan.build(case["n"], case["q"], case["path"], seed=case["fold_seed"])
    from paper_1608_01398_b200.model_select import LAST_BATCH

    LAST_BATCH.clear()
    rep = gi.cv_iht(view, case["y"], plan, gi.IhtConfig(k=int(case["path"].max())),
                    std_mode=case["std_mode"], warm_start=False)
    # the fits' sweeps really were shared: several residuals per sweep
    assert LAST_BATCH["sweeps"] > 0 and LAST_BATCH["rhs"] >= 2 * LAST_BATCH["sweeps"], LAST_BATCH
    assert rep.k_best == case["k_best"]
    np.testing.assert_allclose(rep.mse, case["mse"], rtol=RTOL)
    np.testing.assert_array_equal(rep.final_model.support, case["final_support"])
    np.testing.assert_allclose(rep.final_model.weights, case["final_weights"], rtol=RTOL,
                               atol=vec_atol(case["final_weights"]))


@pytest.mark.parametrize("name", [k for k in FITS if LARGE[k]["covar_raw"].size == 0])
def test_large_path_lockstep_matches_reference(name, monkeypatch):
    """A model-size path whose budgets run in one lock-step group (one
    tensor-core sweep per round of refreshes) reproduces the golden fits."""
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200.iht import BatchGroup

    monkeypatch.setenv("GI_BATCH", "1")
    case = LARGE[name]
    m = _matrix(case)
    view = gi.StandardizedView(m, gi.CovariateBlock.build(None, n=case["n"]))
    ks = [int(case["k"]), int(case["k"]) + 3, max(1, int(case["k"]) - 2)]
    res = gi.fit_path(view, case["y"], sorted(ks))
    got = res[sorted(ks).index(int(case["k"]))]
    np.testing.assert_array_equal(got.model.support, case["support"])
    assert got.iterations == case["iterations"] and got.reason == case["reason"]
    np.testing.assert_allclose(got.model.weights, case["weights"], rtol=RTOL,
                               atol=vec_atol(case["weights"]))
    np.testing.assert_allclose(got.loss_trace, case["loss_trace"], rtol=RTOL, atol=1e-12)
    with BatchGroup(m) as group:  # stats are reported
        assert group.stats() == (0, 0)
