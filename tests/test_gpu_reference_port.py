"""The reference's own unit tests, ported to the device package.

Each test names the reference test it follows (pkg/tests/<file>:<line>).  Only
tests whose subject is on the hot path are ported; the reference's
DenseDesign-based solver tests run here on packed genotypes with the same
assertions where the property is generic (monotone descent, budget, planted
recovery), and against the oracle otherwise.
"""
import threading
import warnings

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _gi():
    import paper_1608_01398_b200 as gi
    return gi


def codes_rng(rng, n, p, missing_rate=0.1):
    return oracle.random_codes(n, p, seed=int(rng.integers(1 << 30)), missing_rate=missing_rate)


def make_view(codes, with_intercept=False, covar=None):
    gi = _gi()
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    block = None
    if with_intercept or covar is not None:
        block = gi.CovariateBlock.build(covar, n=m.n, add_intercept=with_intercept)
    return gi.StandardizedView(m, block)


def reference_standardized(codes):
    return oracle.OraclePacked.from_codes(codes).decompress(np.arange(codes.shape[1]))


# ------------------------------------------------ test_geno_matrix.py ports
def test_column_stats_hand_example():  # test_geno_matrix.py:22-27
    gi = _gi()
    m = gi.PackedGenotypeMatrix.from_codes(np.array([[0], [0], [3], [3]], np.uint8))
    u, v = gi.column_stats(m)
    assert u[0] == pytest.approx(1.0)
    assert v[0] == pytest.approx(1.0 / np.std([0.0, 0.0, 2.0, 2.0], ddof=1))


def test_all_missing_and_monomorphic_columns():  # :30-41
    gi = _gi()
    m = gi.PackedGenotypeMatrix.from_codes(np.full((6, 1), 1, np.uint8))
    assert m.u[0] == 0.0 and m.v[0] == 0.0
    m = gi.PackedGenotypeMatrix.from_codes(np.full((8, 1), 2, np.uint8))
    assert m.u[0] == 1.0 and m.v[0] == 0.0


def test_column_stats_require_two_samples():  # :52-55
    gi = _gi()
    m = gi.PackedGenotypeMatrix.from_codes(np.array([[0, 2]], np.uint8))
    with pytest.raises(ValueError, match="two samples"):
        gi.column_stats(m)


def test_ax_zero_model_and_single_column(rng):  # :66-75
    gi = _gi()
    codes = codes_rng(rng, 20, 50, 0.15)
    view = make_view(codes)
    model = gi.SparseModel.from_parts([], [], np.zeros(0), k=0, p=50)
    np.testing.assert_array_equal(gi.ax(view, model), np.zeros(20))
    ref = reference_standardized(codes)
    for j in (0, 7, 31):
        got = view.genotypes.ax_columns(np.array([j]), np.array([1.0]))
        np.testing.assert_allclose(got, ref[:, j], atol=1e-12)


def test_ax_index_out_of_range_and_aty_dimension(rng):  # :98-100, :126-128
    gi = _gi()
    view = make_view(codes_rng(rng, 20, 50))
    with pytest.raises(IndexError):
        view.genotypes.ax_columns(np.array([50]), np.array([1.0]))
    with pytest.raises(ValueError):
        gi.aty(view, np.zeros(21))


def test_aty_zero_residual_and_monomorphic_component(rng):  # :105-116
    gi = _gi()
    view = make_view(codes_rng(rng, 20, 50))
    np.testing.assert_array_equal(gi.aty(view, np.zeros(20)), np.zeros(50))
    codes = codes_rng(rng, 12, 4, 0.0)
    codes[:, 2] = 2
    view = make_view(codes)
    r = rng.standard_normal(12)
    r -= r.mean()
    assert gi.aty(view, r)[2] == 0.0
    assert view.genotypes.aty_genetic(r, mode="fast")[2] == 0.0


def test_adjoint_identity(rng):  # :131-142
    gi = _gi()
    codes = codes_rng(rng, 25, 30, 0.1)
    view = make_view(codes, with_intercept=True, covar=rng.standard_normal((25, 2)))
    a = rng.standard_normal(25)
    b = rng.standard_normal(view.total)
    lhs = sum(b[j] * float(a @ gi.ax_parts(view, np.array([j]), np.array([1.0])))
              for j in range(view.p))
    lhs += float(a @ (view.covariates.values @ b[view.p:]))
    rhs = float(b @ gi.aty(view, a))
    assert abs(lhs - rhs) <= 1e-8 * max(abs(rhs), 1.0)


def test_decompress_cases(rng):  # :147-184
    gi = _gi()
    view = make_view(codes_rng(rng, 20, 50))
    assert gi.decompress_active(view, np.array([], np.int64)).shape == (20, 0)
    view1 = make_view(np.array([[0], [2], [3], [2]], np.uint8))
    col = gi.decompress_active(view1, np.array([0]))[:, 0]
    assert col.mean() == pytest.approx(0.0, abs=1e-12)
    assert col.var(ddof=1) == pytest.approx(1.0, rel=1e-12)
    codes = codes_rng(rng, 15, 6, 0.0)
    covar = rng.standard_normal((15, 2))
    view2 = make_view(codes, with_intercept=True, covar=covar)
    out = gi.decompress_active(view2, np.array([1, 4, 6, 8]))
    np.testing.assert_array_equal(out[:, 2], np.ones(15))
    np.testing.assert_allclose(out[:, 3], view2.covariates.values[:, 2])
    codes = codes_rng(rng, 40, 12, 0.0)
    view3 = make_view(codes)
    out = gi.decompress_active(view3, np.arange(12))
    live = view3.genotypes.v > 0
    assert np.abs(out.mean(axis=0)[live]).max() <= 1e-10
    assert np.abs(out[:, live].var(axis=0, ddof=1) - 1.0).max() <= 1e-8


def test_subset_rows_and_with_stats(rng):  # :234-250
    gi = _gi()
    codes = codes_rng(rng, 30, 8, 0.1)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    rows = np.arange(0, 30, 2)
    sub = m.subset_rows(rows)
    ref = oracle.OraclePacked.from_codes(codes[rows])
    np.testing.assert_allclose(sub.u, ref.u, atol=1e-12)
    np.testing.assert_allclose(sub.v, ref.v, atol=1e-12)
    np.testing.assert_array_equal(sub.to_codes(), codes[rows])
    u = np.linspace(0, 2, 8)
    v = np.linspace(0, 1, 8)
    other = m.with_stats(u, v)
    np.testing.assert_array_equal(other.u, u)
    np.testing.assert_array_equal(other.data, m.data)
    with pytest.raises(ValueError):
        m.with_stats(u[:3], v)


def test_mutual_transpose_invariant(rng):  # :209-212
    gi = _gi()
    m = gi.PackedGenotypeMatrix.from_codes(codes_rng(rng, 20, 50, 0.15))
    cols = gi.unpack_codes(m.data, m.n)
    rows = gi.unpack_codes(m.data_t, m.p)
    np.testing.assert_array_equal(cols.T, rows)


def test_concurrent_fits_share_one_matrix(rng):  # :282-304
    gi = _gi()
    codes = codes_rng(rng, 60, 40, 0.05)
    view = make_view(codes, with_intercept=True)
    ys = [rng.standard_normal(60) for _ in range(6)]
    sequential = [gi.fit(view, y, gi.IhtConfig(k=3)).model for y in ys]
    threaded = [None] * len(ys)

    def work(i):
        threaded[i] = gi.fit(view, ys[i], gi.IhtConfig(k=3)).model

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(ys))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for a, b in zip(sequential, threaded):
        np.testing.assert_array_equal(a.support, b.support)
        np.testing.assert_array_equal(a.weights, b.weights)  # bitwise: deterministic kernels


# ------------------------------------------------------- test_iht.py ports
def test_accepted_steps_never_increase_loss(rng):  # test_iht.py:154-162
    gi = _gi()
    for _ in range(10):
        codes = codes_rng(rng, 30, 60, 0.05)
        view = make_view(codes, with_intercept=True)
        support = np.sort(rng.choice(60, 4, replace=False))
        y = view.genotypes.ax_columns(support, rng.standard_normal(4)) \
            + rng.normal(0, 0.3, 30)
        res = gi.fit(view, y, gi.IhtConfig(k=int(rng.integers(1, 9))))
        assert np.diff(res.loss_trace).max(initial=-np.inf) <= 1e-12


def test_fit_never_exceeds_budget_and_zero_budget(rng):  # :212-220, :352-356
    gi = _gi()
    for _ in range(6):
        view = make_view(codes_rng(rng, 40, 30, 0.1), with_intercept=True)
        k = int(rng.integers(0, 6))
        assert gi.fit(view, rng.standard_normal(40), gi.IhtConfig(k=k)).model.nnz <= k
    view = make_view(codes_rng(rng, 20, 6, 0.0))
    res = gi.fit(view, rng.standard_normal(20), gi.IhtConfig(k=0))
    assert res.converged and res.model.nnz == 0


def test_fit_loss_matches_residual_recomputation(rng):  # :222-232
    gi = _gi()
    codes = codes_rng(rng, 40, 25, 0.1)
    view = make_view(codes, with_intercept=True)
    y = rng.standard_normal(40)
    cfg = gi.IhtConfig(k=4)
    state = gi.initial_state(view, y, cfg)
    for _ in range(5):
        gi.iht_step(state, view, y, cfg)
    resid = y - gi.ax_parts(view, state.support, state.beta_gen[state.support], state.beta_cov)
    assert state.loss == pytest.approx(0.5 * float(resid @ resid), rel=1e-8)


def test_fit_covariates_survive_projection(rng):  # :235-242
    gi = _gi()
    codes = codes_rng(rng, 60, 30, 0.0)
    covar = rng.standard_normal((60, 2))
    view = make_view(codes, with_intercept=True, covar=covar)
    y = 2.0 + 1.5 * view.covariates.values[:, 1] + rng.normal(0, 0.1, 60)
    res = gi.fit(view, y, gi.IhtConfig(k=2))
    assert res.model.covar.size == 3
    assert abs(res.model.covar[1]) > 0.5


def test_gradient_matches_finite_differences(rng):  # :245-270
    gi = _gi()
    codes = codes_rng(rng, 15, 20, 0.1)
    view = make_view(codes, with_intercept=True)
    y = rng.standard_normal(15)
    warm = gi.project_sparse(rng.standard_normal(20) * 0.5, 5, covar=rng.standard_normal(1))
    state = gi.initial_state(view, y, gi.IhtConfig(k=5), warm=warm)

    def loss_at(bg, bc):
        sup = np.flatnonzero(bg)
        resid = y - gi.ax_parts(view, sup, bg[sup], bc)
        return 0.5 * float(resid @ resid)

    h = 1e-5
    grad = state.gradient
    for idx in range(view.total):
        bp, cp = state.beta_gen.copy(), state.beta_cov.copy()
        bm, cm = state.beta_gen.copy(), state.beta_cov.copy()
        if idx < view.p:
            bp[idx] += h
            bm[idx] -= h
        else:
            cp[idx - view.p] += h
            cm[idx - view.p] -= h
        numeric = (loss_at(bp, cp) - loss_at(bm, cm)) / (2 * h)
        # the fast X^T r kernel is accurate to ~1e-7 of rms(g)
        assert numeric == pytest.approx(grad[idx], rel=1e-5, abs=1e-6)


def test_fit_rejects_bad_response(rng):  # :273-278
    gi = _gi()
    view = make_view(codes_rng(rng, 10, 4))
    with pytest.raises(ValueError):
        gi.fit(view, np.full(10, np.nan), gi.IhtConfig(k=1))
    with pytest.raises(ValueError):
        gi.fit(view, np.zeros(9), gi.IhtConfig(k=1))


def test_refit_cases(rng):  # :292-349
    gi = _gi()
    codes = codes_rng(rng, 20, 5, 0.0)
    view = make_view(codes, with_intercept=True)
    y = rng.standard_normal(20)
    model = gi.refit_least_squares(view, y, np.array([], np.int64))
    assert model.covar[0] == pytest.approx(float(y.mean()), rel=1e-12)
    assert model.nnz == 0
    codes = codes_rng(rng, 50, 30, 0.05)
    view = make_view(codes, with_intercept=True)
    y = rng.standard_normal(50)
    support = np.sort(rng.choice(30, 6, replace=False))
    model = gi.refit_least_squares(view, y, support)
    a = np.hstack([gi.decompress_active(view, support), view.covariates.values])
    expected = np.linalg.solve(a.T @ a, a.T @ y)
    np.testing.assert_allclose(np.concatenate([model.dense_genetic()[support], model.covar]),
                               expected, rtol=1e-8, atol=1e-10)
    resid = y - gi.ax(view, model)
    assert np.abs(a.T @ resid).max() < 1e-8
    codes = codes_rng(rng, 30, 6, 0.0)
    codes[:, 4] = codes[:, 2]
    view = make_view(codes)
    with pytest.warns(gi.RankDeficientWarning):
        model = gi.refit_least_squares(view, rng.standard_normal(30), np.array([2, 4]))
    assert 2 in model.support and 4 not in model.support
    view = make_view(codes_rng(rng, 10, 20, 0.0), with_intercept=True)
    with pytest.raises(ValueError, match="sample count"):
        gi.refit_least_squares(view, np.zeros(10), np.arange(12))


# ----------------------------------------------- test_model_select.py ports
def planted(seed, n, p, support, weights, noise_sd=0.0, intercept=True):
    codes = oracle.random_codes(n, p, seed=seed)
    view = make_view(codes, with_intercept=intercept)
    y = view.genotypes.ax_columns(np.array(support), np.array(weights))
    if noise_sd > 0:
        y = y + np.random.default_rng(seed + 1).normal(0.0, noise_sd, n)
    return view, y


def test_cv_recovers_planted_budget_noiseless():  # test_model_select.py:64-72
    gi = _gi()
    view, y = planted(42, 150, 80, [10, 40, 71], [1.0, -1.2, 0.9])
    rep = gi.cv_iht(view, y, gi.CvPlan.build(150, 5, np.arange(1, 9), seed=3), gi.IhtConfig(k=8))
    assert rep.k_best == 3
    np.testing.assert_array_equal(rep.final_model.support, [10, 40, 71])


def test_cv_pure_noise_prefers_smallest_budget():  # :75-88
    gi = _gi()
    hits, curves = 0, []
    for seed in range(20):
        codes = oracle.random_codes(100, 50, seed=100 + seed)
        view = make_view(codes, with_intercept=True)
        y = np.random.default_rng(200 + seed).standard_normal(100)
        rep = gi.cv_iht(view, y, gi.CvPlan.build(100, 5, np.arange(1, 11), seed=seed),
                        gi.IhtConfig(k=10))
        hits += rep.k_best == 1
        curves.append(rep.mean_mse)
    assert hits >= 11
    avg = np.mean(curves, axis=0)
    assert avg[-1] > avg[0]


def test_cv_single_perfect_predictor():  # :91-98
    gi = _gi()
    codes = oracle.random_codes(40, 1, seed=5)
    view = make_view(codes, with_intercept=True)
    y = gi.decompress_active(view, np.array([0]))[:, 0]
    rep = gi.cv_iht(view, y, gi.CvPlan.build(40, 2, np.array([1]), seed=1),
                    gi.IhtConfig(k=1, tol=1e-8))
    assert rep.mean_mse[0] < 1e-10 and rep.k_best == 1


def test_cv_training_never_touches_test_rows():  # :119-139
    gi = _gi()
    view, y = planted(12, 60, 30, [4, 17], [1.0, -1.0], noise_sd=0.1)
    plan = gi.CvPlan.build(60, 3, np.array([2]), seed=4)
    train = np.flatnonzero(plan.fold_labels != 1)
    sub = gi.StandardizedView(view.genotypes.subset_rows(train),
                              view.covariates.subset_rows(train))
    a = gi.fit(sub, y[train], gi.IhtConfig(k=2))
    y2 = y.copy()
    y2[plan.fold_labels == 1] += 100.0
    b = gi.fit(sub, y2[train], gi.IhtConfig(k=2))
    np.testing.assert_array_equal(a.model.support, b.model.support)
    np.testing.assert_array_equal(a.model.weights, b.model.weights)


def test_cv_warm_and_global_modes():  # :142-162
    gi = _gi()
    view, y = planted(21, 300, 60, [5, 25, 45], [1.0, -1.0, 0.8], noise_sd=0.05)
    plan = gi.CvPlan.build(300, 5, np.arange(1, 9), seed=6)
    cold = gi.cv_iht(view, y, plan, gi.IhtConfig(k=8), warm_start=False)
    warm = gi.cv_iht(view, y, plan, gi.IhtConfig(k=8), warm_start=True)
    assert cold.k_best == warm.k_best
    np.testing.assert_array_equal(cold.final_model.support, warm.final_model.support)
    np.testing.assert_allclose(warm.mean_mse, cold.mean_mse, rtol=0.25)
    view, y = planted(31, 100, 40, [3, 30], [1.0, -1.0])
    rep = gi.cv_iht(view, y, gi.CvPlan.build(100, 4, np.arange(1, 6), seed=7),
                    gi.IhtConfig(k=5), std_mode="global")
    assert rep.k_best == 2
    np.testing.assert_array_equal(rep.final_model.support, [3, 30])


def test_predict_cases(rng):  # :167-199
    gi = _gi()
    codes = codes_rng(rng, 12, 6, 0.0)
    view = make_view(codes, with_intercept=True)
    model = gi.SparseModel.from_parts([], [], np.array([2.5]), k=0, p=6)
    np.testing.assert_allclose(gi.predict(view, model), np.full(12, 2.5))
    empty = gi.StandardizedView(view.genotypes.subset_rows(np.array([], np.int64)),
                                view.covariates.subset_rows(np.array([], np.int64)))
    assert gi.predict(empty, gi.SparseModel.from_parts([1], [1.0], np.array([0.5]), 1, 6)).size == 0
    codes = codes_rng(rng, 25, 15, 0.1)
    view = make_view(codes, with_intercept=True)
    model = gi.SparseModel.from_parts([2, 9], [0.7, -1.1], np.array([0.3]), k=2, p=15)
    expected = reference_standardized(codes)[:, [2, 9]] @ np.array([0.7, -1.1]) + 0.3
    np.testing.assert_allclose(gi.predict(view, model), expected, atol=1e-10)
    with pytest.raises(ValueError):
        gi.predict(view, gi.SparseModel.from_parts([1], [1.0], np.array([0.5]), k=1, p=7))


def test_cv_requires_packed_genotypes(rng):  # model_select.py:85-86
    gi = _gi()
    from paper_1608_01398_b200.model_select import FoldGenotypes
    view = make_view(codes_rng(rng, 30, 10), with_intercept=True)
    fold_view = gi.StandardizedView(FoldGenotypes(view.genotypes, np.arange(20)),
                                    view.covariates.subset_rows(np.arange(20)))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with pytest.raises(TypeError, match="packed genotypes"):
            gi.cv_iht(fold_view, np.zeros(20), gi.CvPlan.build(20, 2, [1], seed=0),
                      gi.IhtConfig(k=1))
