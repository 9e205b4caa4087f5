"""PLINK BED <-> device loader.

``read_bed`` streams a variant-major BED file straight into a device-resident
``PackedGenotypeMatrix``: the file is read in chunks (never whole in host
memory), each chunk is staged through pinned memory and re-laid out on the
device, and the statistics are computed once at the end.  With ``snp_range``
only one SNP block is read (one GPU's shard).  Unlike the reference
(plink_io.py:82-100 -> geno_matrix.py:281-292) no dense code matrix and no
sample-major copy are built.  ``write_bed`` streams the bytes back (kept
verbatim, padding bits included, so a read/write round trip is byte-identical
as in the reference).  Header checks and messages follow plink_io.py:31-56.
BIM/FAM text parsing stays on the host and is out of scope here.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native
from ._native import check, lib, ptr
from .geno_matrix import PackedGenotypeMatrix, _Handle

BED_MAGIC = bytes([0x6C, 0x1B])
BED_MODE_VARIANT_MAJOR = 0x01
_CHUNK_BYTES = 256 << 20


class PlinkFormatError(ValueError):
    """Malformed BED content (reference plink_io.py:31-32)."""


def _check_header(raw: bytes) -> None:
    if len(raw) < 3:
        raise PlinkFormatError("BED file shorter than its 3-byte header")
    if raw[:2] != BED_MAGIC:
        raise PlinkFormatError(
            f"bad BED magic bytes {raw[0]:#04x} {raw[1]:#04x}; expected 0x6c 0x1b")
    if raw[2] == 0x00:
        raise PlinkFormatError("sample-major BED files (mode 0x00) are not supported; "
                               "re-export in variant-major order")
    if raw[2] != BED_MODE_VARIANT_MAJOR:
        raise PlinkFormatError(f"unknown BED storage mode byte {raw[2]:#04x}")


def bed_record_bytes(n_samples: int) -> int:
    return (n_samples + 3) // 4


def read_bed(path, n_samples: int, n_variants: int, device: int = 0,
             snp_range: tuple[int, int] | None = None) -> PackedGenotypeMatrix:
    """Read a variant-major BED file (or SNPs [j0, j1) of it) onto ``device``."""
    if n_samples < 1:
        raise PlinkFormatError("BED files need at least one sample")
    _native.require_device(device)
    nb = bed_record_bytes(n_samples)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        _check_header(fh.read(3))
        expected = n_variants * nb
        found = size - 3
        if found != expected:
            raise PlinkFormatError(
                f"{path}: expected {expected} data bytes for {n_variants} variants x "
                f"{n_samples} samples, found {found}; BED disagrees with BIM/FAM counts")
        j0, j1 = (0, n_variants) if snp_range is None else (int(snp_range[0]), int(snp_range[1]))
        if not 0 <= j0 <= j1 <= n_variants:
            raise ValueError("SNP range out of bounds")
        out = ctypes.c_void_p(0)
        check(lib().gi_matrix_create(n_samples, j1 - j0, device, ctypes.byref(out)))
        handle = _Handle(out.value)
        per_chunk = max(1, _CHUNK_BYTES // max(nb, 1))
        fh.seek(3 + j0 * nb)
        done = 0
        while done < j1 - j0:
            cnt = min(per_chunk, j1 - j0 - done)
            buf = np.frombuffer(fh.read(cnt * nb), dtype=np.uint8)
            if buf.size != cnt * nb:
                raise PlinkFormatError(f"{path}: truncated BED data")
            check(lib().gi_matrix_upload_bed(handle.raw, done, cnt, ptr(buf)))
            done += cnt
    check(lib().gi_matrix_finalize(handle.raw))
    return PackedGenotypeMatrix(handle, n_samples, j1 - j0, device)


def write_bed(matrix: PackedGenotypeMatrix, path) -> None:
    """Variant-major BED file of the matrix bytes (reference plink_io.py:103-112)."""
    if matrix.n < 1:
        raise ValueError("cannot write a genotype matrix with no samples")
    nb = bed_record_bytes(matrix.n)
    per_chunk = max(1, _CHUNK_BYTES // max(nb, 1))
    with open(path, "wb") as fh:
        fh.write(BED_MAGIC + bytes([BED_MODE_VARIANT_MAJOR]))
        for j0 in range(0, matrix.p, per_chunk):
            cnt = min(per_chunk, matrix.p - j0)
            buf = np.empty((cnt, nb), np.uint8)
            check(lib().gi_matrix_read_bed(matrix.handle, j0, cnt, ptr(buf)))
            fh.write(buf.tobytes())
