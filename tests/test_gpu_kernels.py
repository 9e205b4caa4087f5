"""GPU parity of the packed-genotype kernels against the oracle and the
reference's golden vectors (bit-exact where the reference is bit-reproducible).
"""
import numpy as np
import pytest

import golden_io
import oracle

pytestmark = pytest.mark.gpu


def _gm():
    import paper_1608_01398_b200 as gi
    return gi


def _pair(case):
    codes = golden_io.codes_for(case)
    ref = oracle.OraclePacked.from_codes(codes)
    assert golden_io.sha(ref.data) == case["data_sha"]
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    return codes, ref, dev


@pytest.mark.parametrize("name", sorted(golden_io.load("kernels")))
def test_kernels_bit_exact_vs_reference(name):
    case = golden_io.load("kernels")[name]
    codes, ref, dev = _pair(case)
    np.testing.assert_array_equal(dev.u, case["u"])
    np.testing.assert_array_equal(dev.v, case["v"])
    np.testing.assert_array_equal(dev.data, ref.data)
    np.testing.assert_array_equal(dev.to_codes(), codes)
    np.testing.assert_array_equal(dev.aty_genetic(case["r"]), case["aty"])
    got_ax = dev.ax_columns(case["support"], case["weights"])
    if 4 * case["support"].size < case["p"]:
        # the reference's column sweep (geno_matrix.py:346-348): same operation order
        np.testing.assert_array_equal(got_ax, case["ax"])
    else:
        # the reference switches to its sample-major sweep (:337-345), which sums
        # the same terms in another order
        np.testing.assert_allclose(got_ax, case["ax"], rtol=1e-13, atol=1e-14)
    np.testing.assert_array_equal(dev.decompress(case["support"]), case["decompress"])


@pytest.mark.parametrize("name", sorted(golden_io.load("kernels")))
def test_fast_aty_tolerance(name):
    # the IHT loop's lookup-table kernel: fp32 tables, fp64 accumulation.
    # Tolerance 2e-6 of rms(g) -- the sensitivity bound below which supports and
    # iteration counts are unchanged, 10x under 2e-5.
    case = golden_io.load("kernels")[name]
    _, ref, dev = _pair(case)
    want = case["aty"]
    got = dev.aty_genetic(case["r"], mode="fast")
    scale = max(np.sqrt(np.mean(want ** 2)), 1e-300)
    assert np.max(np.abs(got - want)) <= 2e-6 * scale + 1e-12


@pytest.mark.parametrize("n,p,miss", [(1, 1, 0.0), (3, 33, 0.3), (511, 64, 0.0), (513, 65, 0.02),
                                      (1030, 700, 0.05), (4099, 3000, 0.0), (20000, 257, 0.01)])
def test_kernels_vs_oracle_shapes(n, p, miss):
    rng = np.random.default_rng(n * 7919 + p)
    codes = oracle.random_codes(n, p, seed=n + p, missing_rate=miss)
    ref = oracle.OraclePacked.from_codes(codes)
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    np.testing.assert_array_equal(dev.u, ref.u)
    np.testing.assert_array_equal(dev.v, ref.v)
    r = rng.standard_normal(n) + 3.0  # uncentred on purpose
    want = ref.aty_genetic(r)
    np.testing.assert_array_equal(dev.aty_genetic(r), want)
    fast = dev.aty_genetic(r, mode="fast")
    scale = max(np.sqrt(np.mean(want ** 2)), 1e-300)
    assert np.max(np.abs(fast - want)) <= 2e-6 * scale + 1e-12
    k = min(p, 17)
    idx = np.sort(rng.choice(p, k, replace=False))
    w = rng.standard_normal(k)
    if 4 * k < p:  # the reference's column-sweep branch (geno_matrix.py:346-348)
        np.testing.assert_array_equal(dev.ax_columns(idx, w), ref.ax_columns(idx, w))
    else:
        np.testing.assert_allclose(dev.ax_columns(idx, w), ref.ax_columns(idx, w),
                                   rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(dev.decompress(idx), ref.decompress(idx))


def test_subset_rows_and_masked_stats():
    rng = np.random.default_rng(5)
    codes = oracle.random_codes(777, 130, seed=3, missing_rate=0.1)
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    rows = np.sort(rng.choice(777, 500, replace=False))
    sub = dev.subset_rows(rows)
    np.testing.assert_array_equal(sub.to_codes(), codes[rows])
    ref = oracle.OraclePacked.from_codes(codes[rows])
    np.testing.assert_array_equal(sub.u, ref.u)
    np.testing.assert_array_equal(sub.v, ref.v)
    keep = np.zeros(777, np.uint8)
    keep[rows] = 1
    u, v = dev.masked_stats(keep)
    np.testing.assert_array_equal(u, ref.u)
    np.testing.assert_array_equal(v, ref.v)


def test_synth_matches_cpu_twin():
    gi = _gm()
    for n, p, miss, j0 in [(1000, 70, 0.0, 0), (517, 45, 0.02, 123)]:
        dev = gi.PackedGenotypeMatrix.synthetic(n, p, seed=1608, missing_rate=miss, j_base=j0)
        np.testing.assert_array_equal(dev.data, oracle.synth_bed(1608, n, j0, p, missing=miss))


def test_with_stats_shares_bytes():
    codes = oracle.random_codes(50, 20, seed=9, missing_rate=0.1)
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    u = np.linspace(0, 2, 20)
    v = np.linspace(0, 1, 20)
    other = dev.with_stats(u, v)
    np.testing.assert_array_equal(other.u, u)
    np.testing.assert_array_equal(other.data, dev.data)
    ref = oracle.OraclePacked.from_codes(codes).with_stats(u, v)
    r = np.random.default_rng(1).standard_normal(50)
    np.testing.assert_array_equal(other.aty_genetic(r), ref.aty_genetic(r))


def test_bed_roundtrip_and_shards(tmp_path):
    # plink_io.py:82-112 semantics: verbatim bytes, header checks, size check
    gi = _gm()
    rng = np.random.default_rng(10001)
    for trial in range(12):
        n = int(rng.integers(1, 41))
        p = int(rng.integers(1, 70))
        codes = rng.integers(0, 4, size=(n, p)).astype(np.uint8)
        path = tmp_path / f"f{trial}.bed"
        path.write_bytes(bytes([0x6C, 0x1B, 0x01]) + oracle.pack_codes(codes.T).tobytes())
        m = gi.read_bed(path, n, p)
        np.testing.assert_array_equal(m.to_codes(), codes)
        ref = oracle.OraclePacked.from_codes(codes)
        np.testing.assert_array_equal(m.u, ref.u)
        np.testing.assert_array_equal(m.v, ref.v)
        gi.write_bed(m, tmp_path / "copy.bed")
        assert (tmp_path / "copy.bed").read_bytes() == path.read_bytes()
        j0, j1 = p // 3, p // 3 + (p + 1) // 2
        shard = gi.read_bed(path, n, p, snp_range=(j0, j1))
        np.testing.assert_array_equal(shard.to_codes(), codes[:, j0:j1])
    bad = tmp_path / "bad.bed"
    bad.write_bytes(bytes([0x6C, 0x1B, 0x00]) + bytes(4))
    with pytest.raises(gi.PlinkFormatError, match="sample-major"):
        gi.read_bed(bad, 4, 4)
    bad.write_bytes(bytes([0x6C, 0x1B, 0x01]) + bytes(3))
    with pytest.raises(gi.PlinkFormatError, match="BED disagrees"):
        gi.read_bed(bad, 4, 4)


@pytest.mark.parametrize("order", ["sorted", "shuffled", "duplicates", "spread"])
def test_subset_rows_any_row_order(order):
    """Device row gather vs codes[rows]: sorted rows (staged source tiles),
    unsorted / duplicated / widely spread rows (global-memory fallback), with
    missing codes, a ragged last tile and a ragged last SNP group."""
    gi = _gm()
    rng = np.random.default_rng(7)
    n, p = 5000, 77
    codes = oracle.random_codes(n, p, seed=3, missing_rate=0.05)
    m = gi.PackedGenotypeMatrix.from_codes(codes)
    if order == "sorted":
        rows = np.sort(rng.choice(n, 3001, replace=False))
    elif order == "shuffled":
        rows = rng.permutation(n)[:2999]
    elif order == "duplicates":
        rows = rng.integers(0, n, 1500)
    else:
        rows = np.concatenate([np.arange(0, 4800, 9), [n - 1, 0, n - 2]])
    sub = m.subset_rows(rows)
    np.testing.assert_array_equal(sub.to_codes(), codes[rows])
    ref = oracle.OraclePacked.from_codes(codes[rows])
    np.testing.assert_array_equal(sub.u, ref.u)
    np.testing.assert_array_equal(sub.v, ref.v)


def test_aty_batched_fold_residuals_with_fold_stats():
    """gi_aty_batched over q fold residuals (zero off the fold) with each
    fold's own statistics: exact mode equals the reference algorithm (oracle)
    bit for bit, fast mode within the fast kernel's tolerance; without stats
    it equals gi_aty on the handle's stats."""
    import dataclasses

    gi = _gm()
    rng = np.random.default_rng(21)
    n, p, q = 1500, 700, 3
    codes = oracle.random_codes(n, p, seed=8, missing_rate=0.04)
    dev = gi.PackedGenotypeMatrix.from_codes(codes)
    ref = oracle.OraclePacked.from_codes(codes)
    labels = gi.make_folds(n, q, seed=4)
    R = np.zeros((q, n))
    U = np.zeros((q, p))
    V = np.zeros((q, p))
    for f in range(q):
        keep = (labels != f).astype(np.uint8)
        R[f, keep == 1] = rng.standard_normal(int(keep.sum()))
        U[f], V[f] = dev.masked_stats(keep)
    exact = dev.aty_batched(R, U, V, mode="exact")
    fast = dev.aty_batched(R, U, V, mode="fast")
    for f in range(q):
        want = dataclasses.replace(ref, u=U[f], v=V[f]).aty_genetic(R[f])
        np.testing.assert_array_equal(exact[f], want)
        rms = np.sqrt(np.mean(want ** 2))
        assert np.max(np.abs(fast[f] - want)) <= 2e-6 * rms
    plain = dev.aty_batched(R, mode="exact")
    for f in range(q):
        np.testing.assert_array_equal(plain[f], dev.aty_genetic(R[f], mode="exact"))
    with pytest.raises(ValueError):
        dev.aty_batched(R[:, :10])
    with pytest.raises(ValueError):
        dev.aty_batched(R, U)


@pytest.mark.parametrize("miss,misslist", [(0.05, "0"), (0.02, "1"), (0.0, "1")])
def test_fast_aty_identical_columns_get_identical_gradients(miss, misslist, monkeypatch):
    """SNPs in perfect LD have identical columns; the reference gives them
    identical gradients, so top-k ties go to the lower index.  The fast kernel
    sums its table entries in an order fixed by the word positions (pairwise
    over aligned blocks), so its X^T r of a column depends only on the
    column's codes -- not on the lane/word order it is visited in."""
    gi = _gm()
    rng = np.random.default_rng(17)
    n, half = 3000, 120
    base = oracle.random_codes(n, half, seed=17, missing_rate=miss)
    perm = rng.permutation(half)
    codes = np.concatenate([base, base[:, perm]], axis=1)  # column half + i == column perm[i]
    monkeypatch.setenv("GI_MISSLIST", misslist)  # "0": 2-bit tiles with missing genotypes
    dev = gi.PackedGenotypeMatrix.from_codes(codes)
    assert dev.xtr_base3 == (misslist == "1")
    assert dev.xtr_missing_list == (miss > 0 and misslist == "1")
    for _ in range(3):
        g = dev.aty_genetic(rng.standard_normal(n), mode="fast")
        np.testing.assert_array_equal(g[half:], g[perm])
    # a fit whose top-k meets such a tie picks the lower index, like the oracle
    y = oracle.OraclePacked.from_codes(codes).ax_columns(np.array([perm[3]]), np.array([2.0]))
    y = y + rng.normal(0, 0.1, n)
    view = gi.StandardizedView(dev, gi.CovariateBlock.build(None, n=n))
    got = gi.fit(view, y, gi.IhtConfig(k=1))
    want = oracle.fit(oracle.OracleView(oracle.OraclePacked.from_codes(codes),
                                        oracle.intercept(n)), y, 1)
    np.testing.assert_array_equal(got.model.support, want.support)
    assert got.model.support[0] == min(perm[3], half + 3)


@pytest.mark.parametrize("n,p", [(1, 1), (5, 33), (639, 40), (640, 64), (641, 65), (1281, 700),
                                 (5000, 3000), (20000, 257)])
def test_base3_copy_xtr(n, p):
    """A matrix without missing genotypes gets the base-3 copy (5 genotypes per
    byte, 640-sample tiles); the fast X^T r over it agrees with the reference
    within the fast kernel's tolerance, like the 2-bit tiles' sweep, and a
    rebuilt copy gives the same bits."""
    rng = np.random.default_rng(n * 31 + p)
    codes = oracle.random_codes(n, p, seed=n + 7 * p, missing_rate=0.0)
    ref = oracle.OraclePacked.from_codes(codes)
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert dev.xtr_base3
    r = rng.standard_normal(n) + 1.5
    want = ref.aty_genetic(r)
    scale = max(np.sqrt(np.mean(want ** 2)), 1e-300)
    g3 = dev.aty_genetic(r, mode="fast")
    assert np.max(np.abs(g3 - want)) <= 2e-6 * scale + 1e-12
    assert dev.set_xtr_base3(False) is False
    g2 = dev.aty_genetic(r, mode="fast")
    assert np.max(np.abs(g2 - want)) <= 2e-6 * scale + 1e-12
    assert dev.set_xtr_base3(True) is True
    np.testing.assert_array_equal(dev.aty_genetic(r, mode="fast"), g3)
    np.testing.assert_array_equal(dev.aty_genetic(r), want)  # exact kernel: 2-bit tiles


def test_base3_copy_with_missing_genotypes_carries_the_list(monkeypatch):
    """One missing genotype: the base-3 copy comes with the missing-genotype
    list (csrc/missing.cu); GI_MISSLIST=0 keeps such a matrix on the 2-bit
    tiles; a fold copy without that row has a plain base-3 copy."""
    codes = oracle.random_codes(700, 90, seed=5, missing_rate=0.0)
    codes[13, 77] = 1  # one missing genotype
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert dev.xtr_base3 and dev.xtr_missing_list
    sub = dev.subset_rows(np.array([i for i in range(700) if i != 13]))
    assert sub.xtr_base3 and not sub.xtr_missing_list
    monkeypatch.setenv("GI_MISSLIST", "0")
    dev0 = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert not dev0.xtr_base3
    assert dev0.set_xtr_base3(True) is False
    r = np.random.default_rng(3).standard_normal(700)
    want = oracle.OraclePacked.from_codes(codes).aty_genetic(r)
    scale = np.sqrt(np.mean(want ** 2))
    for m in (dev, dev0):
        assert np.max(np.abs(m.aty_genetic(r, mode="fast") - want)) <= 2e-6 * scale + 1e-12


def test_base3_copy_env_switch(monkeypatch):
    """GI_BASE3=0 keeps X^T r on the 2-bit tiles (read when a matrix is built)."""
    codes = oracle.random_codes(900, 70, seed=11, missing_rate=0.0)
    monkeypatch.setenv("GI_BASE3", "0")
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert not dev.xtr_base3
    monkeypatch.delenv("GI_BASE3")
    dev2 = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert dev2.xtr_base3
    r = np.random.default_rng(2).standard_normal(900)
    want = oracle.OraclePacked.from_codes(codes).aty_genetic(r)
    scale = np.sqrt(np.mean(want ** 2))
    for m in (dev, dev2):
        assert np.max(np.abs(m.aty_genetic(r, mode="fast") - want)) <= 2e-6 * scale + 1e-12


@pytest.mark.parametrize("n,p,miss", [(1, 1, 0.5), (5, 33, 0.04), (511, 31, 0.03), (512, 32, 0.02),
                                      (641, 65, 0.02), (1281, 700, 0.01), (5000, 3000, 0.02),
                                      (20000, 257, 0.03), (3000, 8000, 0.001)])
def test_missing_list_xtr(n, p, miss):
    """X^T r of a matrix with missing genotypes over the base-3 copy plus the
    missing-genotype list (csrc/missing.cu): within the fast kernel's
    tolerance of the reference, close to the 2-bit tiles' sweep, and the same
    bits on every call (the list sums are exact integers)."""
    rng = np.random.default_rng(n * 13 + p)
    codes = oracle.random_codes(n, p, seed=n + 3 * p, missing_rate=miss)
    codes[n - 1, p - 1] = 1  # the last sample of the last SNP
    codes[:, 0] = 1  # an all-missing column
    if p > 2:
        codes[: n // 2, 1] = 1
    ref = oracle.OraclePacked.from_codes(codes)
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    rate = float(np.mean(codes == 1))
    assert dev.xtr_missing_list == (rate <= 0.05)
    for shift in (0.0, 1.5, -40.0):
        r = rng.standard_normal(n) + shift
        want = ref.aty_genetic(r)
        scale = max(np.sqrt(np.mean(want ** 2)), 1e-300)
        got = dev.aty_genetic(r, mode="fast")
        assert np.max(np.abs(got - want)) <= 2e-6 * scale + 1e-12
        np.testing.assert_array_equal(dev.aty_genetic(r, mode="fast"), got)
    if dev.xtr_missing_list:
        dev.set_xtr_base3(False)  # the 2-bit tiles' lookup-table sweep
        g2 = dev.aty_genetic(r, mode="fast")
        assert np.max(np.abs(g2 - got)) <= 2e-6 * scale + 1e-12
        assert dev.set_xtr_base3(True) and dev.xtr_missing_list
        np.testing.assert_array_equal(dev.aty_genetic(r, mode="fast"), got)


def test_missing_list_above_five_percent_stays_on_2bit_tiles():
    codes = oracle.random_codes(2000, 300, seed=2, missing_rate=0.08)
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert not dev.xtr_base3 and not dev.xtr_missing_list


def test_missing_list_tile_overflow_path():
    """Missing genotypes concentrated in one sample tile (every SNP missing on
    the first 512 samples, 2.5% overall): that tile's entries overflow the
    missing-sum kernel's staging buffer and are read from global memory
    (csrc/missing.cu), with the same results as the staged tiles."""
    n, p = 512 * 40, 3000
    codes = oracle.random_codes(n, p, seed=77, missing_rate=0.0)
    codes[:512, :] = 1
    dev = _gm().PackedGenotypeMatrix.from_codes(codes)
    assert dev.xtr_missing_list
    ref = oracle.OraclePacked.from_codes(codes)
    r = np.random.default_rng(8).standard_normal(n) + 0.3
    want = ref.aty_genetic(r)
    scale = np.sqrt(np.mean(want ** 2))
    got = dev.aty_genetic(r, mode="fast")
    assert np.max(np.abs(got - want)) <= 2e-6 * scale + 1e-12
    dev.set_xtr_base3(False)
    g2 = dev.aty_genetic(r, mode="fast")
    assert np.max(np.abs(g2 - want)) <= 2e-6 * scale + 1e-12
