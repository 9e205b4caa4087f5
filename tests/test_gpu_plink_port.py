"""The reference's BED codec tests (pkg/tests/test_plink_io.py:16-186), ported to
the device loader: read_bed streams straight into a device-resident matrix and
write_bed streams it back.  BIM/FAM text parsing is host I/O outside the hot
path and is not ported.  The independent writer is the oracle's packing."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _gi():
    import paper_1608_01398_b200 as gi
    return gi


def write_bytes(path, payload):
    path.write_bytes(payload)
    return path


def reference_bed_bytes(codes):
    return bytes([0x6C, 0x1B, 0x01]) + oracle.OraclePacked.from_codes(codes).data.tobytes()


def test_read_bed_decodes_standard_code_table(tmp_path):  # :16-24
    gi = _gi()
    bed = write_bytes(tmp_path / "one.bed", bytes([0x6C, 0x1B, 0x01, 0b11100100]))
    matrix = gi.read_bed(bed, n_samples=4, n_variants=1)
    dosage = matrix.to_dosage()[:, 0]
    assert dosage[0] == 0.0
    assert np.isnan(dosage[1])
    assert dosage[2] == 1.0
    assert dosage[3] == 2.0


def test_read_bed_empty_variant_file(tmp_path):  # :27-32
    gi = _gi()
    bed = write_bytes(tmp_path / "empty.bed", bytes([0x6C, 0x1B, 0x01]))
    matrix = gi.read_bed(bed, n_samples=4, n_variants=0)
    assert matrix.p == 0 and matrix.n == 4 and matrix.u.size == 0


def test_roundtrip_against_independent_writer(tmp_path):  # :35-43
    gi = _gi()
    codes = oracle.random_codes(50, 100, seed=35, missing_rate=0.1)
    payload = reference_bed_bytes(codes)
    matrix = gi.read_bed(write_bytes(tmp_path / "ref.bed", payload), n_samples=50,
                         n_variants=100)
    np.testing.assert_array_equal(matrix.to_codes(), codes)
    out = tmp_path / "copy.bed"
    gi.write_bed(matrix, out)
    assert out.read_bytes() == payload


def test_write_bed_single_byte_example_and_padding(tmp_path):  # :46-59
    gi = _gi()
    out = tmp_path / "w.bed"
    gi.write_bed(gi.PackedGenotypeMatrix.from_codes(np.array([[0], [1], [2], [3]], np.uint8)), out)
    assert out.read_bytes() == bytes([0x6C, 0x1B, 0x01, 0b11100100])
    gi.write_bed(gi.PackedGenotypeMatrix.from_codes(np.full((5, 1), 3, np.uint8)), out)
    assert out.read_bytes() == bytes([0x6C, 0x1B, 0x01, 0b11111111, 0b00000011])


def test_write_read_roundtrip_13x7_and_snp_range(tmp_path):  # :62-68
    gi = _gi()
    codes = oracle.random_codes(13, 7, seed=62, missing_rate=0.2)
    out = tmp_path / "rt.bed"
    gi.write_bed(gi.PackedGenotypeMatrix.from_codes(codes), out)
    np.testing.assert_array_equal(gi.read_bed(out, 13, 7).to_codes(), codes)
    # a rank's SNP block of the same file (the multi-GPU loader)
    np.testing.assert_array_equal(gi.read_bed(out, 13, 7, snp_range=(2, 5)).to_codes(),
                                  codes[:, 2:5])


@pytest.mark.parametrize("payload,n,p,match", [
    (bytes([0x00, 0x1B, 0x01, 0x00]), 4, 1, "magic"),          # :79-82
    (bytes([0x6C, 0x1B, 0x00, 0x00]), 4, 1, "sample-major"),   # :85-88
    (bytes([0x6C, 0x1B, 0x02, 0x00]), 4, 1, "mode"),           # :91-94
    (bytes([0x6C, 0x1B, 0x01, 0x00]), 4, 2, "BIM/FAM"),        # :97-100
])
def test_malformed_bed_rejected(tmp_path, payload, n, p, match):
    gi = _gi()
    with pytest.raises(gi.PlinkFormatError, match=match):
        gi.read_bed(write_bytes(tmp_path / "bad.bed", payload), n, p)


def test_stats_from_packed_match_decoded_dense():  # :179-186
    gi = _gi()
    codes = oracle.random_codes(30, 40, seed=179, missing_rate=0.2)
    matrix = gi.PackedGenotypeMatrix.from_codes(codes)
    dose = np.where(codes == 1, np.nan, np.select([codes == 2, codes == 3], [1.0, 2.0], 0.0))
    u_ref = np.nan_to_num(np.nanmean(dose, axis=0))
    sd = np.nanstd(dose, axis=0, ddof=1)
    v_ref = np.where(sd > 0, 1.0 / np.where(sd > 0, sd, 1.0), 0.0)
    np.testing.assert_allclose(matrix.u, u_ref, atol=1e-12)
    np.testing.assert_allclose(matrix.v, v_ref, atol=1e-12)
