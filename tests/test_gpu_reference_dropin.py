"""The UNMODIFIED reference package on the B200.

genoiht 0.1.0 is installed verbatim into baseline/_ref (pip --target, no
source change).  These tests put a device-resident
PackedGenotypeMatrix into the reference's OWN StandardizedView and
CovariateBlock and call the reference's own functions:

* operator protocol, no dispatch: genoiht.aty / ax / decompress_active and a
  whole genoiht.fit run their kernels on the GPU and equal the reference's
  CPU results BIT FOR BIT (the device operators reproduce _aty_kernel,
  _ax_cols_kernel and _decompress_kernel exactly; geno_matrix.py:142-236);
* with the two-line dispatch of INTEGRATION.md installed at run time
  (paper_1608_01398_b200.integration.install): genoiht.fit and
  genoiht.cv_iht -- unchanged call sites -- run the native device loop and
  match the reference's CPU fit / CV (support, iterations, k_best exact;
  beta, loss, MSE within 1e-6 relative).
Skipped, visibly, when baseline/_ref is absent.
"""
import os
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
RTOL = 1e-6


@pytest.fixture(scope="module")
def genoiht():
    if not os.path.isdir(os.path.join(REF, "genoiht")):
        pytest.skip("baseline/_ref not installed (pip install --no-deps --target baseline/_ref "
                    "<reference pkg>)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/genoiht_numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import genoiht as g
    assert g.__file__.startswith(REF)
    return g


def _pair(genoiht, n, p, seed, miss):
    import paper_1608_01398_b200 as gi

    data = oracle.synth_bed(seed, n, 0, p, missing=miss)
    cpu = genoiht.PackedGenotypeMatrix.from_bed_buffer(data, n)
    dev = gi.PackedGenotypeMatrix.from_bed_buffer(data, n)
    return cpu, dev


def _views(genoiht, cpu, dev, n, cov_raw=None):
    block = genoiht.CovariateBlock.build(cov_raw, n=n)
    return genoiht.StandardizedView(cpu, block), genoiht.StandardizedView(dev, block)


def test_reference_operators_on_device_are_bit_identical(genoiht):
    n, p = 1500, 8000
    cpu, dev = _pair(genoiht, n, p, 91, 0.02)
    np.testing.assert_array_equal(dev.u, cpu.u)
    np.testing.assert_array_equal(dev.v, cpu.v)
    v_cpu, v_dev = _views(genoiht, cpu, dev, n)
    r = np.random.default_rng(1).standard_normal(n)
    np.testing.assert_array_equal(genoiht.aty(v_dev, r), genoiht.aty(v_cpu, r))
    model = genoiht.SparseModel.from_parts(np.array([3, 77, 4000]), np.array([0.5, -1.0, 2.0]),
                                           np.array([0.25]), k=3, p=p)
    np.testing.assert_array_equal(genoiht.ax(v_dev, model), genoiht.ax(v_cpu, model))
    sup = np.array([5, 6, 7999, p])  # the last index pulls the covariate column
    np.testing.assert_array_equal(genoiht.decompress_active(v_dev, sup),
                                  genoiht.decompress_active(v_cpu, sup))


def test_reference_fit_loop_over_device_operators_is_bit_identical(genoiht):
    """No dispatch: the reference's own Python loop (iht.py:326-354), every
    X^T r / X_S w / decompress on the GPU -- the same FitResult, bit for bit."""
    n, p = 1200, 5000
    cpu, dev = _pair(genoiht, n, p, 92, 0.03)
    v_cpu, v_dev = _views(genoiht, cpu, dev, n)
    y, _ = genoiht.simulate_phenotype(v_cpu, genoiht.SimulationSpec(k_true=6, seed=3))
    cfg = genoiht.IhtConfig(k=8)
    want = genoiht.fit(v_cpu, y, cfg)
    got = genoiht.fit(v_dev, y, cfg)
    np.testing.assert_array_equal(got.model.support, want.model.support)
    np.testing.assert_array_equal(got.model.weights, want.model.weights)
    np.testing.assert_array_equal(got.loss_trace, want.loss_trace)
    assert got.iterations == want.iterations and got.reason == want.reason


def test_cv_without_dispatch_is_refused_by_the_reference(genoiht):
    """Why cv_iht needs the dispatch: the reference's _fold_views accepts
    only its own matrix class (model_select.py:85-86)."""
    n, p = 300, 500
    cpu, dev = _pair(genoiht, n, p, 93, 0.0)
    _, v_dev = _views(genoiht, cpu, dev, n)
    plan = genoiht.CvPlan.build(n, 3, np.arange(1, 4), seed=1)
    with pytest.raises(TypeError):
        genoiht.cv_iht(v_dev, np.zeros(n), plan, genoiht.IhtConfig(k=3))


@pytest.fixture
def dispatched(genoiht):
    from paper_1608_01398_b200 import integration

    integration.install(genoiht)
    yield genoiht
    integration.uninstall(genoiht)


@pytest.mark.parametrize("miss,cov", [(0.0, False), (0.02, True)])
def test_reference_fit_dispatches_to_native_loop(dispatched, miss, cov):
    from paper_1608_01398_b200.iht import last_native_fit_info

    genoiht = dispatched
    n, p = 3000, 16000  # fast X^T r kernel (> 2 MiB of tiles)
    cpu, dev = _pair(genoiht, n, p, 94, miss)
    raw = np.random.default_rng(5).standard_normal((n, 2)) if cov else None
    v_cpu, v_dev = _views(genoiht, cpu, dev, n, raw)
    y, _ = genoiht.simulate_phenotype(v_cpu, genoiht.SimulationSpec(k_true=12, seed=4))
    cfg = genoiht.IhtConfig(k=15)
    want = genoiht.fit(v_cpu, y, cfg)  # the reference's own loop on the host
    got = genoiht.fit(v_dev, y, cfg)   # unchanged call site -> device loop
    assert last_native_fit_info()["xtr_kernel"].startswith("fast"), last_native_fit_info()
    np.testing.assert_array_equal(got.model.support, want.model.support)
    assert got.iterations == want.iterations and got.reason == want.reason
    atol = RTOL * float(np.max(np.abs(want.model.weights)))
    np.testing.assert_allclose(got.model.weights, want.model.weights, rtol=RTOL, atol=atol)
    np.testing.assert_allclose(got.model.covar, want.model.covar, rtol=RTOL, atol=1e-12)
    np.testing.assert_allclose(got.loss_trace, want.loss_trace, rtol=RTOL)


@pytest.mark.parametrize("std_mode", ["train", "global"])
def test_reference_cv_dispatches_to_device(dispatched, std_mode):
    genoiht = dispatched
    n, p = 1500, 9000
    cpu, dev = _pair(genoiht, n, p, 95, 0.01)
    v_cpu, v_dev = _views(genoiht, cpu, dev, n)
    y, _ = genoiht.simulate_phenotype(v_cpu, genoiht.SimulationSpec(k_true=5, seed=6))
    plan = genoiht.CvPlan.build(n, 4, np.arange(1, 9), seed=2016)
    cfg = genoiht.IhtConfig(k=8)
    want = genoiht.cv_iht(v_cpu, y, plan, cfg, std_mode=std_mode)
    got = genoiht.cv_iht(v_dev, y, plan, cfg, std_mode=std_mode)
    assert got.k_best == want.k_best
    np.testing.assert_allclose(got.mse, want.mse, rtol=RTOL)
    np.testing.assert_array_equal(got.final_model.support, want.final_model.support)
    atol = RTOL * float(np.max(np.abs(want.final_model.weights)))
    np.testing.assert_allclose(got.final_model.weights, want.final_model.weights, rtol=RTOL,
                               atol=atol)


def _report_eq(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g.k_true, g.snr_divisor, g.replicate) == (w.k_true, w.snr_divisor, w.replicate)
        assert g.k_selected == w.k_selected
        assert (g.precision, g.recall) == (w.precision, w.recall)
        for f in ("mse_test", "h2_true", "h2_est"):
            np.testing.assert_allclose(getattr(g, f), getattr(w, f), rtol=RTOL)


GRID = dict(k_true_grid=[3, 6], snr_divisors=[1.0, 4.0], replicates=2, q=3, path_points=5,
            seed=11)


def test_device_run_experiment_matches_reference(genoiht):
    """The experiment grid (reference simulate.py:123-186) on the device --
    paper_1608_01398_b200.run_experiment -- against the reference's own on
    the host: same selected budgets, precision and recall; MSE and h^2 within
    1e-6."""
    import paper_1608_01398_b200 as gi

    n, p = 700, 2400
    cpu, dev = _pair(genoiht, n, p, 96, 0.01)
    want = genoiht.run_experiment(genoiht.StandardizedView(cpu, genoiht.CovariateBlock.build(
        None, n=n)), config=genoiht.IhtConfig(k=12), **GRID)
    got = gi.run_experiment(gi.StandardizedView(dev, gi.CovariateBlock.build(None, n=n)),
                            config=gi.IhtConfig(k=12), **GRID)
    _report_eq(got, want)
    rows_g, rows_w = gi.aggregate_reports(got), genoiht.aggregate_reports(want)
    assert [r["k_true"] for r in rows_g] == [r["k_true"] for r in rows_w]
    for a, b in zip(rows_g, rows_w):
        np.testing.assert_allclose(a["precision"], b["precision"])
        np.testing.assert_allclose(a["mse"], b["mse"], rtol=RTOL)


def test_reference_run_experiment_on_device_matrix(dispatched):
    """The reference's OWN run_experiment, unchanged, over a device matrix
    (its subset_rows / with_stats / cv_iht / predict / heritability reach the
    B200 through the operator protocol and the installed dispatch)."""
    genoiht = dispatched
    n, p = 700, 2400
    cpu, dev = _pair(genoiht, n, p, 97, 0.0)
    block = genoiht.CovariateBlock.build(None, n=n)
    want = genoiht.run_experiment(genoiht.StandardizedView(cpu, block),
                                  config=genoiht.IhtConfig(k=12), **GRID)
    got = genoiht.run_experiment(genoiht.StandardizedView(dev, block),
                                 config=genoiht.IhtConfig(k=12), **GRID)
    _report_eq(got, want)
