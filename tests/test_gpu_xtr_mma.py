"""The tensor-core X^T R kernel (csrc/xtr_mma.cu, tcgen05.mma kind::i8).

Checked against the reference's _aty_kernel as restated by the oracle
(bit-exact to the reference's golden vectors, tests/test_oracle.py): the
kernel's sums are exact integers of the residual quantised to 2^-26 of its
largest centred value, so its error is the quantisation's alone -- bounded
here at 2e-7 of rms(g) (typically ~2e-8), 10x inside the 2e-6 rms(g) the
survey found supports and iteration counts stable under.
Covers missing genotypes, ragged n (partial tiles and bytes) and p (partial
M-tiles of 128 SNPs), every batch width (1..32 right-hand sides: MMA N = 8 ..
128) and per-RHS statistics (CV folds standardised with their training rows).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

TOL = 2e-7


def _pair(n, p, seed, miss):
    import paper_1608_01398_b200 as gi

    codes = oracle.random_codes(n, p, seed=seed, missing_rate=miss)
    return gi.PackedGenotypeMatrix.from_codes(codes), oracle.OraclePacked.from_codes(codes)


def _check(got, want):
    rms = float(np.sqrt(np.mean(want ** 2))) or 1.0
    err = float(np.max(np.abs(got - want))) / rms
    assert err <= TOL, f"max error {err:.3g} of rms(g)"
    return err


@pytest.mark.parametrize("n,p,miss", [(1000, 10000, 0.0), (1000, 10000, 0.02), (777, 333, 0.05),
                                      (4097, 1029, 0.0), (130, 129, 0.1), (5, 40, 0.3),
                                      (20000, 3000, 0.01)])
def test_mma_single_rhs_matches_reference_kernel(n, p, miss):
    m, ref = _pair(n, p, seed=n + p, miss=miss)
    rng = np.random.default_rng(n)
    r = rng.standard_normal(n) * 3.0 + 0.7  # off-centre: the epilogue restores the mean
    _check(m.aty_genetic(r, mode="mma"), ref.aty_genetic(r))


@pytest.mark.parametrize("B", [1, 2, 3, 4, 5, 8, 9, 12, 13, 16, 17, 20, 21, 32, 33, 40])
@pytest.mark.parametrize("miss", [0.0, 0.02])
def test_mma_batched_matches_per_rhs_reference(B, miss):
    n, p = 2500, 4000
    m, ref = _pair(n, p, seed=B, miss=miss)
    rng = np.random.default_rng(B + 100)
    R = rng.standard_normal((B, n)) * rng.uniform(0.1, 10.0, (B, 1))
    R[:, rng.random(n) < 0.2] = 0.0  # fold-like zeros
    G = m.aty_batched(R, mode="mma")
    for b in range(B):
        _check(G[b], ref.aty_genetic(R[b]))


def test_mma_batched_with_fold_stats():
    """Each right-hand side under its own (training-fold) statistics, as the
    CV folds use them: equals the reference kernel on with_stats(u_f, v_f)."""
    n, p, q = 3000, 2000, 5
    m, ref = _pair(n, p, seed=9, miss=0.02)
    rng = np.random.default_rng(9)
    labels = rng.permutation(n) % q
    R = np.zeros((q, n))
    U = np.zeros((q, p))
    V = np.zeros((q, p))
    for f in range(q):
        keep = labels != f
        U[f], V[f] = m.masked_stats(keep.astype(np.uint8))
        R[f, keep] = rng.standard_normal(int(keep.sum()))
    G = m.aty_batched(R, U, V, mode="mma")
    for f in range(q):
        fold_ref = oracle.OraclePacked(n=n, p=p, data=ref.data, u=U[f], v=V[f])
        _check(G[f], fold_ref.aty_genetic(R[f]))


def test_mma_identical_columns_get_identical_gradients():
    """Integer sums are order-free: duplicated SNP columns (perfect LD) in
    different lanes, groups and M-tiles get bit-identical gradients, so the
    reference's lower-index tie rule sees the same ties."""
    import paper_1608_01398_b200 as gi

    n = 3333
    base = oracle.random_codes(n, 7, seed=3, missing_rate=0.03)
    cols = [0, 1, 2, 3, 4, 5, 6] * 60  # copies spread over lanes, groups, M-tiles
    codes = np.ascontiguousarray(base[:, cols])
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    r = np.random.default_rng(4).standard_normal(n)
    g = m.aty_genetic(r, mode="mma")
    for c in range(7):
        vals = g[np.arange(c, len(cols), 7)]
        assert np.all(vals == vals[0])


def test_mma_zero_and_constant_residuals():
    m, ref = _pair(600, 300, seed=1, miss=0.05)
    np.testing.assert_array_equal(m.aty_genetic(np.zeros(600), mode="mma"), np.zeros(300))
    # a constant residual has g = 0 up to rounding (the reference's own sums
    # leave ~1e-13): compared absolutely
    r = np.full(600, 2.5)
    np.testing.assert_allclose(m.aty_genetic(r, mode="mma"), ref.aty_genetic(r), rtol=0,
                               atol=1e-9)
