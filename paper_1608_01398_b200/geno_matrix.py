"""Device-resident packed genotype matrices behind the reference operator protocol.

Mirrors the public surface of ``genoiht.geno_matrix`` (reference
/root/reference/pkg/src/genoiht/geno_matrix.py) for the IHT hot path:
``PackedGenotypeMatrix`` keeps the 2-bit genotypes in B200 HBM (swizzled sample
tiles, csrc/common.cuh) and implements the protocol the solver uses --
``n``, ``p``, ``u``, ``v``, ``aty_genetic``, ``ax_columns``, ``decompress``,
``subset_rows``, ``with_stats``, ``to_codes`` -- through the C ABI of
libgenoiht_cuda.so.  ``CovariateBlock``, ``StandardizedView``, ``ax_parts``,
``ax``, ``aty`` and ``decompress_active`` keep the reference's semantics.

Every genotype operation runs on the GPU; nothing falls back to the CPU.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import check, lib, ptr

CODE_HOM_A1 = 0  # dosage 0
CODE_MISSING = 1
CODE_HET = 2  # dosage 1
CODE_HOM_A2 = 3  # dosage 2
_DOSE_OF_CODE = np.array([0.0, 0.0, 1.0, 2.0])


def set_worker_threads(count: int) -> int:
    """API parity with geno_matrix.set_worker_threads (:64-73).

    Device kernels have no host worker pool; results never depend on this
    value.  Returns the effective (clamped) count like the reference.
    """
    return max(1, int(count))


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """(rows, cols) 2-bit codes -> (rows, ceil(cols/4)) bytes, first entry in the
    least significant bit pair, zero padding (reference :76-89)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    rows, cols = codes.shape
    nb = (cols + 3) // 4
    wide = np.zeros((rows, 4 * nb), np.uint8)
    wide[:, :cols] = codes
    q = wide.reshape(rows, nb, 4)
    return np.ascontiguousarray(q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4)
                                | (q[:, :, 3] << 6), dtype=np.uint8)


def unpack_codes(packed: np.ndarray, length: int) -> np.ndarray:
    """Inverse of pack_codes (reference :92-103)."""
    packed = np.asarray(packed, dtype=np.uint8)
    rows, nb = packed.shape
    if length > 4 * nb:
        raise ValueError(f"cannot unpack {length} entries from {nb} bytes per row")
    out = np.empty((rows, 4 * nb), np.uint8)
    for slot in range(4):
        out[:, slot::4] = (packed >> (2 * slot)) & 3
    return np.ascontiguousarray(out[:, :length])


_ATY_MODES = {"exact": 0, "fast": 1, "mma": 2}


def _aty_mode(mode: str) -> int:
    try:
        return _ATY_MODES[mode]
    except KeyError:
        raise ValueError(f"unknown X^T r mode {mode!r} (exact, fast or mma)") from None


class _Handle:
    """Owns one gi_matrix*; freed when the last Python reference goes away."""

    def __init__(self, raw: int):
        self.raw = ctypes.c_void_p(raw)

    def __del__(self):
        try:
            if self.raw:
                lib().gi_matrix_free(self.raw)
                self.raw = ctypes.c_void_p(0)
        except Exception:  # interpreter shutdown
            pass


def _new_handle(fn, *args) -> _Handle:
    out = ctypes.c_void_p(0)
    check(fn(*args, ctypes.byref(out)))
    return _Handle(out.value)


class PackedGenotypeMatrix:
    """2-bit genotype matrix resident on a B200, with cached standardisation stats.

    Drop-in for genoiht's PackedGenotypeMatrix (geno_matrix.py:249-373).  The
    packed bytes live on ``device`` only; ``data`` (the reference's
    variant-major buffer) and ``data_t`` are materialised on demand.
    ``u``/``v`` are per-SNP means and inverse standard deviations over
    non-missing entries, bit-identical to the reference (v = 0 for monomorphic
    or all-missing columns).
    """

    def __init__(self, handle: _Handle, n: int, p: int, device: int,
                 u: np.ndarray | None = None, v: np.ndarray | None = None):
        self._h = handle
        self.n = int(n)
        self.p = int(p)
        self.device = int(device)
        self._u = u
        self._v = v
        self._data = None
        self._lock = threading.Lock()

    # ---------------------------------------------------------- constructors
    @classmethod
    def from_bed_buffer(cls, data: np.ndarray, n_samples: int, device: int = 0):
        """From a raw (p, ceil(n/4)) variant-major byte buffer, kept verbatim
        (reference :281-292)."""
        _native.require_device(device)
        data = np.ascontiguousarray(data, dtype=np.uint8)
        if data.ndim != 2:
            raise ValueError("BED buffer must be a 2-d (variants, bytes) array")
        n = int(n_samples)
        if data.shape[1] != (n + 3) // 4:
            raise ValueError("BED buffer width does not match the sample count")
        h = _new_handle(lib().gi_matrix_from_bed, ptr(data), n, data.shape[0], device)
        return cls(h, n, data.shape[0], device)

    @classmethod
    def from_codes(cls, codes: np.ndarray, device: int = 0):
        """From an (n, p) array of 2-bit genotype codes (reference :267-279)."""
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        if codes.ndim != 2:
            raise ValueError("codes must be a 2-d array of samples x variants")
        if codes.size and codes.max() > 3:
            raise ValueError("genotype codes must lie in {0, 1, 2, 3}")
        n, p = codes.shape
        return cls.from_bed_buffer(pack_codes(codes.T).reshape(p, (n + 3) // 4), n,
                                   device=device)

    @classmethod
    def synthetic(cls, n: int, p: int, seed: int, maf_range=(0.05, 0.5),
                  missing_rate: float = 0.0, device: int = 0, j_base: int = 0):
        """Generate genotypes on the device (law of simulate.random_packed_matrix,
        simulate.py:56-65; counter-based stream, CPU twin in oracle/)."""
        _native.require_device(device)
        h = _new_handle(lib().gi_matrix_synth, ctypes.c_uint64(int(seed) & (2**64 - 1)), int(n),
                        int(p), int(j_base), float(maf_range[0]), float(maf_range[1]),
                        float(missing_rate), device)
        return cls(h, n, p, device)

    # ------------------------------------------------------------ attributes
    is_cuda = True  # lets a patched genoiht.fit / cv_iht dispatch to the device loop

    def _fetch_stats(self):
        with self._lock:
            if self._u is None:
                u = np.zeros(self.p)
                v = np.zeros(self.p)
                if self.p:
                    check(lib().gi_matrix_stats(self._h.raw, ptr(u), ptr(v)))
                u.setflags(write=False)
                v.setflags(write=False)
                self._u, self._v = u, v

    @property
    def u(self) -> np.ndarray:
        self._fetch_stats()
        return self._u

    @property
    def v(self) -> np.ndarray:
        self._fetch_stats()
        return self._v

    @property
    def handle(self):
        return self._h.raw

    @property
    def data(self) -> np.ndarray:
        """Variant-major BED bytes uint8[p, ceil(n/4)] (downloaded once)."""
        with self._lock:
            if self._data is None:
                nb = (self.n + 3) // 4
                out = np.zeros((self.p, nb), np.uint8)
                if self.p and nb:
                    check(lib().gi_matrix_read_bed(self._h.raw, 0, self.p, ptr(out)))
                out.setflags(write=False)
                self._data = out
            return self._data

    @property
    def data_t(self) -> np.ndarray:
        """Sample-major packing of the transpose (reference keeps it resident;
        here it is derived on request -- the device path never needs it)."""
        return pack_codes(self.to_codes())

    @property
    def nbytes_packed(self) -> int:
        return self.p * ((self.n + 3) // 4) + self.n * ((self.p + 3) // 4)

    @property
    def missing_counts(self) -> np.ndarray:
        out = np.zeros(self.p, np.int32)
        if self.p:
            check(lib().gi_matrix_missing_counts(self._h.raw, ptr(out)))
        return out

    @property
    def xtr_base3(self) -> bool:
        """True when X^T r streams the device's base-3 copy (5 genotypes per
        byte, csrc/layout.cu; with missing genotypes, beside their position
        list, csrc/missing.cu)."""
        out = ctypes.c_int(0)
        check(lib().gi_matrix_xtr_format(self._h.raw, -1, ctypes.byref(out)))
        return bool(out.value)

    @property
    def xtr_missing_list(self) -> bool:
        """True when X^T r takes the missing sums from the missing-genotype
        list (a matrix with missing genotypes on the base-3 copy)."""
        out = ctypes.c_int(0)
        check(lib().gi_matrix_xtr_format(self._h.raw, -1, ctypes.byref(out)))
        return out.value == 2

    def set_xtr_base3(self, enable: bool) -> bool:
        """Build (when possible) or drop the base-3 copy; returns xtr_base3.
        Shared with with_stats copies of this matrix."""
        out = ctypes.c_int(0)
        check(lib().gi_matrix_xtr_format(self._h.raw, 1 if enable else 0, ctypes.byref(out)))
        return bool(out.value)

    def to_codes(self) -> np.ndarray:
        return np.ascontiguousarray(unpack_codes(self.data, self.n).T)

    def to_dosage(self) -> np.ndarray:
        codes = self.to_codes()
        out = _DOSE_OF_CODE[codes]
        out[codes == CODE_MISSING] = np.nan
        return out

    # --------------------------------------------------------- derived views
    def subset_rows(self, rows) -> "PackedGenotypeMatrix":
        """Rows gathered on the device; u and v recomputed (reference :305-308)."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        if rows.size and (rows.min() < 0 or rows.max() >= self.n):
            raise IndexError("sample index out of range")
        h = _new_handle(lib().gi_matrix_subset_rows, self._h.raw, ptr(rows), rows.size)
        return PackedGenotypeMatrix(h, rows.size, self.p, self.device)

    def with_stats(self, u, v) -> "PackedGenotypeMatrix":
        """Same packed bytes, caller-supplied stats (reference :310-316)."""
        u = np.array(u, dtype=np.float64)
        v = np.array(v, dtype=np.float64)
        if u.shape != (self.p,) or v.shape != (self.p,):
            raise ValueError("stats vectors must have one entry per variant")
        h = _new_handle(lib().gi_matrix_with_stats, self._h.raw, ptr(u), ptr(v))
        out = PackedGenotypeMatrix(h, self.n, self.p, self.device)
        u.setflags(write=False)
        v.setflags(write=False)
        out._u, out._v = u, v
        return out

    def with_masked_stats(self, keep) -> "PackedGenotypeMatrix":
        """Same packed bytes standardised with the statistics of the rows with
        keep != 0 (what subset_rows(rows) would compute), formed on the device;
        u / v are downloaded only if read."""
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        if keep.shape != (self.n,):
            raise ValueError("row mask must have one entry per sample")
        h = _new_handle(lib().gi_matrix_with_masked_stats, self._h.raw, ptr(keep))
        return PackedGenotypeMatrix(h, self.n, self.p, self.device)

    def masked_stats(self, keep) -> tuple[np.ndarray, np.ndarray]:
        """u, v over the rows with keep != 0 -- what subset_rows(rows) would
        compute, without materialising the subset."""
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        if keep.shape != (self.n,):
            raise ValueError("row mask must have one entry per sample")
        u = np.zeros(self.p)
        v = np.zeros(self.p)
        if self.p:
            check(lib().gi_matrix_masked_stats(self._h.raw, ptr(keep), ptr(u), ptr(v)))
        return u, v

    # -------------------------------------------------------------- protocol
    def _check_index(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        if idx.size and (idx.min() < 0 or idx.max() >= self.p):
            raise IndexError("variant index out of range")
        return idx

    def ax_columns(self, idx, w) -> np.ndarray:
        """sum_t w[t] * standardized column idx[t]; bit-identical to the
        reference's column sweep (geno_matrix.py:168-194)."""
        idx = self._check_index(idx)
        w = np.ascontiguousarray(w, dtype=np.float64)
        if w.shape != idx.shape:
            raise ValueError("index and weight vectors must align")
        out = np.zeros(self.n)
        if idx.size == 0 or self.n == 0:
            return out
        check(lib().gi_ax_cols(self._h.raw, ptr(idx), ptr(w), idx.size, ptr(out)))
        return out

    def aty_genetic(self, r, mode: str = "exact") -> np.ndarray:
        """Standardized X^T r over every column (reference :351-364).

        mode="exact" reproduces _aty_kernel bit-for-bit; mode="fast" is the
        lookup-table kernel (relative error ~1e-7); mode="mma" the tensor-core
        kernel over exact integer sums of the quantised residual (~1e-8)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        if r.shape != (self.n,):
            raise ValueError(f"residual vector must have length {self.n}")
        out = np.empty(self.p)
        if self.p == 0:
            return out
        if self.n == 0:
            out[:] = 0.0
            return out
        check(lib().gi_aty(self._h.raw, ptr(r), float(r.sum()), ptr(out), _aty_mode(mode)))
        return out

    def aty_batched(self, R, U=None, V=None, mode: str = "exact") -> np.ndarray:
        """aty_genetic for each row of R (B, n) -- e.g. CV fold residuals, zero
        off the fold -- optionally under per-row stats U, V (B, p); returns
        (B, p).  Row b equals aty_genetic(R[b]) on with_stats(U[b], V[b]),
        bit for bit in exact mode.  One device call (gi_aty_batched); in
        mode="mma" every batch of up to 32 residuals (16 when genotypes are
        missing) is ONE sweep of the matrix on the tensor cores."""
        R = np.ascontiguousarray(np.atleast_2d(R), dtype=np.float64)
        if R.ndim != 2 or R.shape[1] != self.n:
            raise ValueError(f"residual matrix must have {self.n} columns")
        B = R.shape[0]
        if (U is None) != (V is None):
            raise ValueError("pass both U and V, or neither")
        if U is not None:
            U = np.ascontiguousarray(U, dtype=np.float64)
            V = np.ascontiguousarray(V, dtype=np.float64)
            if U.shape != (B, self.p) or V.shape != (B, self.p):
                raise ValueError("stats matrices must be (batch, variants)")
        out = np.zeros((B, self.p))
        if self.p == 0 or self.n == 0 or B == 0:
            return out
        sums = np.array([float(r.sum()) for r in R])
        check(lib().gi_aty_batched(self._h.raw, ptr(R), ptr(sums),
                                   None if U is None else ptr(U), None if V is None else ptr(V),
                                   B, ptr(out), _aty_mode(mode)))
        return out

    def decompress(self, idx) -> np.ndarray:
        """Dense standardized (n, k) submatrix (reference :366-373)."""
        idx = self._check_index(idx)
        out_t = np.zeros((idx.size, self.n))
        if idx.size and self.n:
            check(lib().gi_decompress(self._h.raw, ptr(idx), idx.size, ptr(out_t)))
        return out_t.T

    def __repr__(self):
        return f"PackedGenotypeMatrix(n={self.n}, p={self.p}, device=cuda:{self.device})"


def column_stats(matrix: PackedGenotypeMatrix) -> tuple[np.ndarray, np.ndarray]:
    """Per-column mean and inverse sd over non-missing entries (reference :376-383)."""
    if matrix.n < 2:
        raise ValueError("column statistics need at least two samples")
    return np.array(matrix.u), np.array(matrix.v)


_PINV_LOCK = threading.Lock()


@dataclass(frozen=True, eq=False)
class CovariateBlock:
    """Dense non-genetic covariates, standardised once; the intercept column is
    all ones (reference :476-518)."""

    values: np.ndarray
    labels: tuple

    @property
    def c(self) -> int:
        return self.values.shape[1]

    @classmethod
    def build(cls, raw=None, n=None, labels=None, add_intercept: bool = True,
              standardize: bool = True) -> "CovariateBlock":
        columns, names = [], []
        if add_intercept:
            if raw is None and n is None:
                raise ValueError("need a sample count to build an intercept column")
            rows = n if raw is None else np.asarray(raw).shape[0]
            columns.append(np.ones(rows))
            names.append("intercept")
        if raw is not None:
            raw = np.asarray(raw, dtype=np.float64)
            if raw.ndim == 1:
                raw = raw[:, None]
            for j in range(raw.shape[1]):
                col = raw[:, j].copy()
                if standardize:
                    sd = col.std(ddof=1) if col.size > 1 else 0.0
                    col = (col - col.mean()) / sd if sd > 0 else col - col.mean()
                columns.append(col)
                names.append(labels[j] if labels is not None else f"covar{j + 1}")
        if not columns:
            raise ValueError("covariate block needs an intercept or data columns")
        return cls(values=np.column_stack(columns), labels=tuple(names))

    def subset_rows(self, rows) -> "CovariateBlock":
        return CovariateBlock(values=self.values[np.asarray(rows)], labels=self.labels)

    def least_squares(self, y) -> np.ndarray:
        """The minimum-norm least-squares coefficients of y on the block -- the
        reference's ``np.linalg.lstsq(C, y, rcond=None)`` (iht.py:208) -- through
        a pseudo-inverse cached on the (immutable) block with lstsq's rank
        cutoff (eps * max(n, c) * sigma_max): one (c, n) x n product per fit
        instead of an SVD of C (2 ms at n = 100k), equal to lstsq's solution up
        to rounding."""
        pinv = self.__dict__.get("_pinv")
        if pinv is None:
            with _PINV_LOCK:  # concurrent first fits on a block compute it once
                pinv = self.__dict__.get("_pinv")
                if pinv is None:
                    n, c = self.values.shape
                    pinv = np.linalg.pinv(self.values,
                                          rtol=np.finfo(np.float64).eps * max(n, c))
                    object.__setattr__(self, "_pinv", pinv)
        # an elementwise product and row sums, not BLAS: fits run concurrently
        # from a thread pool (cv_iht, fit_path), and concurrent multithreaded
        # GEMV calls oversubscribe the host cores (CV 0.43 -> 0.67 s)
        return np.multiply(pinv, np.asarray(y, dtype=np.float64)).sum(axis=1)


@dataclass(frozen=True, eq=False)
class StandardizedView:
    """Genetic predictors (indices < p) followed by covariates (indices >= p)
    (reference :521-550)."""

    genotypes: object
    covariates: CovariateBlock | None = None

    def __post_init__(self):
        if self.covariates is not None and self.covariates.values.shape[0] != self.genotypes.n:
            raise ValueError("covariate rows must match the sample count")

    @property
    def n(self) -> int:
        return self.genotypes.n

    @property
    def p(self) -> int:
        return self.genotypes.p

    @property
    def c(self) -> int:
        return 0 if self.covariates is None else self.covariates.c

    @property
    def total(self) -> int:
        return self.p + self.c


def ax_parts(view: StandardizedView, support, weights, covar=None) -> np.ndarray:
    """X_st b + C b_cov (reference :553-562)."""
    out = view.genotypes.ax_columns(support, weights)
    if covar is not None and view.c:
        covar = np.asarray(covar, dtype=np.float64)
        if covar.shape != (view.c,):
            raise ValueError("covariate coefficient length mismatch")
        out = out + view.covariates.values @ covar
    return out


def ax(view: StandardizedView, model) -> np.ndarray:
    return ax_parts(view, model.support, model.weights, model.covar)


def aty(view: StandardizedView, r) -> np.ndarray:
    """X^T r over genetic predictors, covariates appended (reference :570-575)."""
    gen = view.genotypes.aty_genetic(r)
    if view.c:
        return np.concatenate([gen, view.covariates.values.T @ np.asarray(r, dtype=np.float64)])
    return gen


def decompress_active(view: StandardizedView, support) -> np.ndarray:
    """Dense standardized (n, k) columns in predictor order; indices >= p pull
    covariate columns (reference :578-592)."""
    support = np.asarray(support, dtype=np.int64)
    if support.size and (support.min() < 0 or support.max() >= view.total):
        raise IndexError("predictor index out of range")
    gen_idx = support[support < view.p]
    cov_idx = support[support >= view.p] - view.p
    out = np.empty((view.n, support.size), order="F")
    out[:, : gen_idx.size] = view.genotypes.decompress(gen_idx)
    if cov_idx.size:
        out[:, gen_idx.size:] = view.covariates.values[:, cov_idx]
    return out
