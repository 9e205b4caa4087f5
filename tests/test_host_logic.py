"""Host-side logic of the drop-in that runs without a GPU: projection and
top-k rules, fold bookkeeping, configuration validation, codes packing and
the per-shard top-k merge.  Cases mirror the reference's own tests
(pkg/tests/test_iht.py:33-69, test_model_select.py:28-61, test_plink_io.py:16-24)."""
import itertools

import numpy as np
import pytest

import oracle
import paper_1608_01398_b200 as gi
from paper_1608_01398_b200.dist import merge_topk, shard_range


def test_project_examples():
    m = gi.project_sparse(np.array([3.0, -1.0, 0.5, 2.0]), 2)
    np.testing.assert_array_equal(m.dense_genetic(), [3.0, 0.0, 0.0, 2.0])
    m = gi.project_sparse(np.array([2.0, -2.0, 0.0]), 1)  # tie -> lower index
    np.testing.assert_array_equal(m.dense_genetic(), [2.0, 0.0, 0.0])
    m = gi.project_sparse(np.array([1.0, -1.0, 1.0]), 3)
    np.testing.assert_array_equal(m.dense_genetic(), [1.0, -1.0, 1.0])


def test_hard_threshold_matches_oracle(rng):
    for _ in range(300):
        p = int(rng.integers(1, 30))
        k = int(rng.integers(0, 8))
        vec = np.round(rng.standard_normal(p), int(rng.integers(0, 3)))  # rounding makes ties
        np.testing.assert_array_equal(gi.hard_threshold(vec, k), oracle.threshold_k(vec, k))


def test_top_k_large(rng):
    vec = rng.standard_normal(200_000)
    idx = gi.top_k_indices(np.abs(vec), 10)
    assert set(idx) == set(np.argsort(-np.abs(vec))[:10])


def test_merge_topk_matches_global_rule(rng):
    # per-shard local top-k lists merged == global top-k with ties to lower index
    for _ in range(200):
        p = int(rng.integers(1, 60))
        k = int(rng.integers(1, 10))
        world = int(rng.integers(1, 5))
        vals = np.round(rng.standard_normal(p), 1)
        vals[rng.random(p) < 0.2] = 0.0
        keys_all = np.abs(vals).view(np.uint64) + np.uint64(1)
        ks, ii, vv = [], [], []
        for r in range(world):
            j0, j1 = shard_range(p, world, r)
            loc = np.arange(j0, j1)
            order = np.lexsort((loc, ~keys_all[loc]))[:k]
            ks.append(keys_all[loc][order])
            ii.append(loc[order])
            vv.append(vals[loc][order])
        idx, got = merge_topk(np.concatenate(ks), np.concatenate(ii), np.concatenate(vv), k)
        want_idx = oracle.top_k(np.abs(vals), k)
        np.testing.assert_array_equal(idx, want_idx)
        np.testing.assert_array_equal(got, vals[want_idx])


def test_shard_range_partitions():
    for p, world in itertools.product([0, 1, 7, 100, 1001], [1, 2, 3, 8]):
        spans = [shard_range(p, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == p
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 == b0
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1


def test_folds_match_reference_rule():
    for n, q, seed in [(10, 5, 0), (7, 3, 0), (40, 4, 9), (2000, 5, 2016)]:
        np.testing.assert_array_equal(gi.make_folds(n, q, seed), oracle.folds(n, q, seed))
    assert np.bincount(gi.make_folds(10, 5, 0)).tolist() == [2] * 5
    with pytest.raises(ValueError):
        gi.make_folds(5, 1, 0)
    with pytest.raises(ValueError):
        gi.make_folds(5, 6, 0)


def test_plan_and_select():
    with pytest.raises(ValueError):
        gi.CvPlan.build(20, 4, [3, 2, 5], seed=0)
    with pytest.raises(ValueError):
        gi.CvPlan.build(20, 4, [0, 1], seed=0)
    path = np.array([2, 4, 6])
    assert gi.select_k(path, np.array([0.5, 0.25, 0.25])) == 4
    assert gi.select_k(path, np.array([0.25, 0.25, 0.25])) == 2


def test_config_validation():
    for bad in (dict(k=-1), dict(k=1, tol=0.0), dict(k=1, c_omega=1.0), dict(k=1, max_iter=0),
                dict(k=1, max_backtracks=-1)):
        with pytest.raises(ValueError):
            gi.IhtConfig(**bad)


def test_sparse_model_rules():
    m = gi.SparseModel.from_parts([5, 1, 3], [0.0, 2.0, -1.0], np.zeros(1), k=3, p=10)
    np.testing.assert_array_equal(m.support, [1, 3])
    with pytest.raises(ValueError):
        gi.SparseModel(support=np.array([3, 1]), weights=np.ones(2), covar=np.zeros(0), k=2, p=5)


def test_pack_codes_kat():
    # the byte 0b11100100 holds codes 0, 1, 2, 3 from the least significant pair
    assert gi.pack_codes(np.array([[0, 1, 2, 3]], np.uint8))[0, 0] == 0b11100100
    codes = np.random.default_rng(3).integers(0, 4, size=(9, 13)).astype(np.uint8)
    np.testing.assert_array_equal(gi.unpack_codes(gi.pack_codes(codes), 13), codes)
    np.testing.assert_array_equal(gi.pack_codes(codes), oracle.pack_codes(codes))


def test_covariate_block():
    raw = np.random.default_rng(2).standard_normal((10, 2)) * 5 + 2
    block = gi.CovariateBlock.build(raw, add_intercept=True)
    np.testing.assert_array_equal(block.values[:, 0], np.ones(10))
    assert block.labels[0] == "intercept"
    np.testing.assert_allclose(block.values[:, 1:].mean(axis=0), 0.0, atol=1e-12)


def test_fit_path_runs_sharded_fits_one_at_a_time(monkeypatch):
    """Sharded views share one communicator per process group, so fit_path
    must not run their fits concurrently (advisor finding, round 1)."""
    import numpy as np

    from paper_1608_01398_b200 import model_select as ms

    seen = {}

    def fake_run(jobs, workers):
        seen["workers"] = workers
        return [(None, None) for _ in jobs]

    class Shard:  # what dist.ShardedGenotypes looks like to fit_path
        n, p = 10, 20
        comm = object()

        def native_comm(self):  # pragma: no cover - never called here
            raise AssertionError

    class View:
        genotypes = Shard()
        n, p, c = 10, 20, 0

    monkeypatch.setattr(ms, "_run_concurrently", fake_run)
    ms.fit_path(View(), np.zeros(10), [1, 2, 3], workers=8)
    assert seen["workers"] == 1


def test_integration_install_dispatches_reference_entry_points(monkeypatch):
    """paper_1608_01398_b200.integration.install(genoiht): the reference's fit
    and cv_iht -- in every module that bound them -- go to the device loop for
    device-resident views and stay the reference's otherwise; uninstall
    restores them (host-side check with a stand-in device matrix)."""
    import os
    import sys

    import numpy as np
    import pytest

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(root, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "genoiht")):
        pytest.skip("baseline/_ref not installed")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/genoiht_numba_cache")
    sys.path.insert(0, ref)
    try:
        import genoiht
        import genoiht.cli
        import genoiht.model_select
        from paper_1608_01398_b200 import iht as dev_iht
        from paper_1608_01398_b200 import integration
        from paper_1608_01398_b200 import model_select as dev_ms

        calls = []
        monkeypatch.setattr(dev_iht, "fit", lambda *a, **k: calls.append("fit") or "device-fit")
        monkeypatch.setattr(dev_ms, "cv_iht", lambda *a, **k: calls.append("cv") or "device-cv")

        class DeviceLike:
            is_cuda = True
            n, p = 4, 3

        ref_fit = genoiht.iht.fit
        view = genoiht.StandardizedView(DeviceLike(), None)
        integration.install(genoiht)
        integration.install(genoiht)  # idempotent
        try:
            assert genoiht.fit(view, np.zeros(4), genoiht.IhtConfig(k=1)) == "device-fit"
            assert genoiht.model_select.fit(view, np.zeros(4), genoiht.IhtConfig(k=1)) == \
                "device-fit"
            assert genoiht.cli.fit is genoiht.fit
            assert genoiht.cv_iht(view, np.zeros(4), None, None) == "device-cv"
            assert calls == ["fit", "fit", "cv"]
            # host views still take the reference path
            codes = np.array([[0, 2, 3], [2, 3, 0], [3, 0, 2], [0, 0, 3]], np.uint8)
            host = genoiht.StandardizedView(genoiht.PackedGenotypeMatrix.from_codes(codes), None)
            res = genoiht.fit(host, np.array([1.0, -1.0, 0.5, 0.0]), genoiht.IhtConfig(k=1))
            assert type(res).__module__ == "genoiht.iht"
        finally:
            integration.uninstall(genoiht)
        assert genoiht.iht.fit is ref_fit and genoiht.fit is ref_fit
        assert genoiht.model_select.fit is ref_fit
    finally:
        sys.path.remove(ref)


def test_simulation_helpers_match_reference_definitions():
    """precision_recall / straddling_path / dense_path (reference
    simulate.py:95-120) on their edge cases."""
    import numpy as np
    import pytest

    import paper_1608_01398_b200 as gi

    assert gi.precision_recall([1, 2, 3], [2, 3, 4]) == (2 / 3, 2 / 3)
    assert gi.precision_recall([], [5]) == (0.0, 0.0)
    with pytest.raises(ValueError, match="non-empty"):
        gi.precision_recall([1], [])
    np.testing.assert_array_equal(gi.straddling_path(3, 5), [1, 3, 5, 7, 9])
    np.testing.assert_array_equal(gi.straddling_path(20, 5, 2), [16, 18, 20, 22, 24])
    np.testing.assert_array_equal(gi.dense_path(2, 3), [1, 2, 3, 4, 5])
