"""The reference's acceptance gate (pkg/tests/test_acceptance.py), ported to
the device package.  Criteria on the hot path, same thresholds:

  01 oracle equivalence on random packed matrices   (:38-59)
  03 monotone descent across seeded fits            (:77-95)
  06 CV budget selection and path-edge saturation   (:160-197)
  07 refit matches the normal equations             (:200-219)
  08 determinism across worker counts               (:222-266; CUDA streams here)
  10 BED codec fuzzed round trips                   (:281-299)

Criteria 02 (host projection), 04 (DenseDesign recovery), 05 (simulation
grid) and 09 (CLI benchmark table) are off the packed-genotype hot path; the
host projection is covered by tests/test_host_logic.py and the benchmark
table by test_gpu_fit.py::test_cli_bench_tables.
"""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _gi():
    import paper_1608_01398_b200 as gi
    return gi


def rel_err(got, want):
    scale = np.linalg.norm(want)
    return float(np.linalg.norm(got - want)) / (scale if scale > 0 else 1.0)


def test_01_oracle_equivalence_on_random_packed_matrices():
    gi = _gi()
    rng = np.random.default_rng(1001)
    worst = worst_fast = 0.0
    for trial in range(200):
        n = int(rng.integers(5, 101))
        p = int(rng.integers(2, 301))
        codes = oracle.random_codes(n, p, seed=trial, missing_rate=float(rng.uniform(0.0, 0.2)))
        matrix = gi.PackedGenotypeMatrix.from_codes(codes)
        dense = oracle.OraclePacked.from_codes(codes).decompress(np.arange(p))  # (n, p)
        r = rng.standard_normal(n)
        k = int(rng.integers(1, min(p, 12) + 1))
        support = np.sort(rng.choice(p, k, replace=False))
        weights = rng.standard_normal(k)
        worst = max(worst,
                    rel_err(matrix.aty_genetic(r), dense.T @ r),
                    rel_err(matrix.ax_columns(support, weights), dense[:, support] @ weights),
                    rel_err(matrix.decompress(support), dense[:, support]))
        worst_fast = max(worst_fast, rel_err(matrix.aty_genetic(r, mode="fast"), dense.T @ r))
    assert worst < 1e-10, f"max rel err {worst:.2e}"
    assert worst_fast < 1e-6, f"fast X^T r max rel err {worst_fast:.2e}"


def test_03_monotone_descent_across_seeded_fits():
    gi = _gi()
    from paper_1608_01398_b200.simulate import random_packed_matrix

    worst = -np.inf
    for seed in range(100):
        rng = np.random.default_rng(2000 + seed)
        matrix = random_packed_matrix(200, 500, seed=3000 + seed)
        view = gi.StandardizedView(matrix, gi.CovariateBlock.build(None, n=200))
        k_true = int(rng.integers(2, 9))
        support = np.sort(rng.choice(500, k_true, replace=False))
        divisor = float(rng.choice([1.0, 2.0, 10.0, 20.0]))
        weights = rng.normal(0.0, np.sqrt(1.0 / divisor), k_true)
        y = gi.ax_parts(view, support, weights) + rng.normal(0.0, 0.1, 200)
        result = gi.fit(view, y, gi.IhtConfig(k=int(rng.integers(1, 13))))
        diffs = np.diff(result.loss_trace)
        if diffs.size:
            worst = max(worst, float(diffs.max()))
    assert worst <= 1e-12, f"max loss increase {worst:.2e}"


def test_06_cv_selects_planted_budget_and_saturates_at_path_edge():
    gi = _gi()
    from paper_1608_01398_b200.simulate import random_packed_matrix

    hits = 0
    for seed in range(20):
        rng = np.random.default_rng(6000 + seed)
        matrix = random_packed_matrix(500, 1000, seed=6500 + seed)
        view = gi.StandardizedView(matrix, gi.CovariateBlock.build(None, n=500))
        support = np.sort(rng.choice(1000, 5, replace=False))
        weights = rng.uniform(0.5, 1.5, 5) * rng.choice([-1.0, 1.0], 5)
        y = gi.ax_parts(view, support, weights)
        plan = gi.CvPlan.build(500, 5, np.arange(1, 16), seed=seed)
        hits += gi.cv_iht(view, y, plan, gi.IhtConfig(k=15)).k_best == 5

    rng = np.random.default_rng(6999)
    matrix = random_packed_matrix(400, 300, seed=6998)
    view = gi.StandardizedView(matrix, gi.CovariateBlock.build(None, n=400))
    support = np.sort(rng.choice(300, 12, replace=False))
    y = gi.ax_parts(view, support, np.ones(12))
    plan = gi.CvPlan.build(400, 5, np.arange(1, 7), seed=1)
    upper_edge = gi.cv_iht(view, y, plan, gi.IhtConfig(k=6)).k_best

    lower_hits = 0
    for seed in range(5):
        rng = np.random.default_rng(6800 + seed)
        matrix = random_packed_matrix(200, 300, seed=6900 + seed)
        noisy = gi.StandardizedView(matrix, gi.CovariateBlock.build(None, n=200))
        support = np.sort(rng.choice(300, 2, replace=False))
        y2 = gi.ax_parts(noisy, support, np.array([1.0, -1.0])) + rng.normal(0, 0.7, 200)
        plan2 = gi.CvPlan.build(200, 5, np.arange(8, 21, 2), seed=seed)
        lower_hits += gi.cv_iht(noisy, y2, plan2, gi.IhtConfig(k=20)).k_best == 8
    assert hits >= 18 and upper_edge == 6 and lower_hits >= 4, \
        f"k_best=5 in {hits}/20; edge {upper_edge}; saturation {lower_hits}/5"


def test_07_refit_matches_normal_equations():
    gi = _gi()
    rng = np.random.default_rng(7001)
    worst = 0.0
    for trial in range(100):
        n = int(rng.integers(30, 80))
        p = int(rng.integers(10, 40))
        codes = oracle.random_codes(n, p, seed=7000 + trial, missing_rate=0.05)
        view = gi.StandardizedView(gi.PackedGenotypeMatrix.from_codes(codes),
                                   gi.CovariateBlock.build(None, n=n))
        k = int(rng.integers(1, min(8, p)))
        support = np.sort(rng.choice(p, k, replace=False))
        support = support[view.genotypes.v[support] > 0]  # skip monomorphic columns
        y = rng.standard_normal(n)
        model = gi.refit_least_squares(view, y, support)
        a = np.hstack([gi.decompress_active(view, support), view.covariates.values])
        expected = np.linalg.solve(a.T @ a, a.T @ y)
        got = np.concatenate([model.dense_genetic()[support], model.covar])
        worst = max(worst, float(np.abs(got - expected).max()))
    assert worst < 1e-8, f"max coefficient deviation {worst:.2e}"


def test_08_byte_identical_outputs_across_worker_counts(monkeypatch):
    """Reference: cv/fit/simulate tables and kernel outputs identical for 1, 2
    and 8 numba threads.  Here the workers are concurrent fits on their own
    CUDA streams; every reduction is deterministic, so the reports and kernel
    outputs must match byte for byte."""
    gi = _gi()
    from paper_1608_01398_b200.simulate import random_packed_matrix

    matrix = random_packed_matrix(800, 2000, seed=8001, missing_rate=0.02)
    view = gi.StandardizedView(matrix, gi.CovariateBlock.build(None, n=800))
    support = np.array([7, 220, 1410])
    y = gi.ax_parts(view, support, np.array([1.0, -1.1, 0.9]))
    y = y + np.random.default_rng(8002).normal(0, 0.05, 800)
    r = np.random.default_rng(8003).standard_normal(800)
    plan = gi.CvPlan.build(800, 4, np.arange(1, 9), seed=11)
    outputs = {}
    for workers in ("1", "2", "8"):
        monkeypatch.setenv("GI_FIT_WORKERS", workers)
        rep = gi.cv_iht(view, y, plan, gi.IhtConfig(k=8))
        path = gi.fit_path(view, y, np.arange(1, 9))
        outputs[workers] = (
            rep.mse.tobytes(), rep.final_model.weights.tobytes(),
            b"".join(res.model.weights.tobytes() + res.loss_trace.tobytes() for res in path),
            gi.aty(view, r).tobytes(),
            matrix.aty_genetic(r, mode="fast").tobytes(),
            gi.ax_parts(view, support, np.ones(3)).tobytes())
    assert outputs["1"] == outputs["2"] == outputs["8"]


def test_10_bed_codec_fuzzed_roundtrips(tmp_path):
    gi = _gi()
    rng = np.random.default_rng(10001)
    checked = {0: 0, 1: 0, 2: 0, 3: 0}
    for trial in range(500):
        n = int(rng.integers(1, 41))
        p = int(rng.integers(0, 30))
        codes = rng.integers(0, 4, size=(n, p)).astype(np.uint8)
        matrix = gi.PackedGenotypeMatrix.from_codes(codes)
        path = tmp_path / f"f{trial % 8}.bed"
        gi.write_bed(matrix, path)
        again = gi.read_bed(path, n, p)
        np.testing.assert_array_equal(again.to_codes(), codes)
        second = tmp_path / "copy.bed"
        gi.write_bed(again, second)
        assert second.read_bytes() == path.read_bytes()
        checked[n % 4] += 1
    assert all(count > 0 for count in checked.values())
