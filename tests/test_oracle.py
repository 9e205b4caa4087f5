"""Pin the CPU oracle against the reference's own outputs (tests/golden).

The oracle (oracle/genoiht_oracle.c + oracle/oracle.py) is a restatement of
genoiht 0.1.0; these tests show it reproduces the reference bit-for-bit on the
kernels and exactly (support, iterations, weights, loss trace) on fits and CV.
"""
import numpy as np
import pytest

import golden_io
import oracle


def _matrix(case):
    codes = golden_io.codes_for(case)
    m = oracle.OraclePacked.from_codes(codes)
    assert golden_io.sha(m.data) == case["data_sha"], "generator drifted from the reference"
    return m


@pytest.mark.parametrize("name", sorted(golden_io.load("kernels")))
def test_oracle_kernels_bit_exact(name):
    case = golden_io.load("kernels")[name]
    m = _matrix(case)
    np.testing.assert_array_equal(m.u, case["u"])
    np.testing.assert_array_equal(m.v, case["v"])
    np.testing.assert_array_equal(m.aty_genetic(case["r"]), case["aty"])
    np.testing.assert_array_equal(m.ax_columns(case["support"], case["weights"]), case["ax"])
    np.testing.assert_array_equal(m.decompress(case["support"]), case["decompress"])
    dense = m.ax_columns(np.arange(m.p), case["dense_w"])
    np.testing.assert_allclose(dense, case["ax_dense"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_thread_invariance(threads):
    case = golden_io.load("kernels")["kernel6"]
    m = _matrix(case)
    oracle.set_threads(threads)
    try:
        np.testing.assert_array_equal(m.aty_genetic(case["r"]), case["aty"])
    finally:
        oracle.set_threads(0)


def _view(case, m):
    return oracle.OracleView(m, oracle.intercept(case["n"]) if case["intercept"] else None)


@pytest.mark.parametrize("name", sorted(golden_io.load("fits")))
def test_oracle_fit_matches_reference(name):
    case = golden_io.load("fits")[name]
    m = _matrix(case)
    res = oracle.fit(_view(case, m), case["y"], int(case["k"]))
    np.testing.assert_array_equal(res.support, case["support"])
    assert res.iterations == case["iterations"]
    assert res.reason == case["reason"]
    np.testing.assert_allclose(res.weights, case["weights"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.covar, case["covar"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(res.loss_trace, case["loss_trace"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("name", sorted(golden_io.load("cv")))
def test_oracle_cv_matches_reference(name):
    case = golden_io.load("cv")[name]
    m = _matrix(case)
    view = oracle.OracleView(m, oracle.intercept(case["n"]))
    labels = oracle.folds(case["n"], case["q"], case["fold_seed"])
    np.testing.assert_array_equal(labels, case["labels"])
    rep = oracle.cv(view, case["y"], case["q"], case["path"], case["fold_seed"],
                    std_mode=case["std_mode"], warm_start=bool(case["warm"]))
    assert rep.k_best == case["k_best"]
    np.testing.assert_allclose(rep.mse, case["mse"], rtol=1e-10, atol=1e-14)
    np.testing.assert_array_equal(rep.final[0], case["final_support"])
    np.testing.assert_allclose(rep.final[1], case["final_weights"], rtol=1e-10)
    np.testing.assert_allclose(rep.final[2], case["final_covar"], rtol=1e-10, atol=1e-14)


def test_synth_twin_distribution():
    # the counter-based generator reproduces the reference's genotype law
    data = oracle.synth_bed(1608, 4000, 0, 300, missing=0.02)
    m = oracle.OraclePacked.from_bed(data, 4000)
    codes = m.to_codes()
    miss = float(np.mean(codes == 1))
    assert 0.017 < miss < 0.023
    assert m.u.min() > 0.0 and m.u.max() < 1.1
    # slices are independent of how the SNP range is cut
    np.testing.assert_array_equal(oracle.synth_bed(1608, 4000, 100, 50, missing=0.02),
                                  data[100:150])


LARGE = golden_io.load("large")


def _large_matrix(case):
    data = oracle.synth_bed(case["seed"], case["n"], 0, case["p"], missing=case["missing"])
    assert golden_io.sha(data) == case["data_sha"], "synthetic-BED twin drifted"
    return oracle.OraclePacked.from_bed(data, case["n"])


@pytest.mark.parametrize("name", sorted(k for k, v in LARGE.items() if v["kind"] == "fit"))
def test_oracle_large_fit_matches_reference(name):
    """The fast-kernel-sized golden fits (tests/test_gpu_large_parity.py):
    the oracle reproduces the reference on them, so the GPU comparison is
    against pinned numbers."""
    from paper_1608_01398_b200.geno_matrix import CovariateBlock

    case = LARGE[name]
    m = _large_matrix(case)
    raw = case["covar_raw"]
    cov = CovariateBlock.build(raw if raw.size else None, n=case["n"]).values
    res = oracle.fit(oracle.OracleView(m, cov), case["y"], int(case["k"]))
    np.testing.assert_array_equal(res.support, case["support"])
    assert res.iterations == case["iterations"] and res.reason == case["reason"]
    np.testing.assert_allclose(res.weights, case["weights"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.loss_trace, case["loss_trace"], rtol=1e-12, atol=1e-15)


def test_oracle_large_cv_matches_reference():
    case = LARGE["cvL_global_warm_miss"]
    m = _large_matrix(case)
    rep = oracle.cv(oracle.OracleView(m, oracle.intercept(case["n"])), case["y"], case["q"],
                    case["path"], case["fold_seed"], std_mode=case["std_mode"],
                    warm_start=bool(case["warm"]))
    assert rep.k_best == case["k_best"]
    np.testing.assert_allclose(rep.mse, case["mse"], rtol=1e-10, atol=1e-14)
    np.testing.assert_array_equal(rep.final[0], case["final_support"])
