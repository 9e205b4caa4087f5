"""Device state and fused phases of one IHT fit on one SNP shard.

The IHT control flow (iht.py) is the reference's, step for step; everything
O(n), O(p) or O(n p) it needs runs as libgenoiht_cuda.so kernels on the
shard's GPU, with only O(k) values crossing to the host once per phase:

    refresh      X_S w (+ all-reduce) -> r = y - X_S w - C b_cov, loss, centred
                 fp32 residual, g = -X^T r (lookup-table kernel), g_cov, max|g|,
                 g on the support                       (iht.py:183-191, :257-261)
    image        ||X_idx w + C w_cov||^2                 (iht.py:238-241, :295-296)
    top-k        k largest |beta - mu g| or |g|          (iht.py:36-58, :228, :280)

``ShardEngine`` holds the sharding and communication logic (global <-> local
SNP indices, which partial products are all-reduced, how per-shard top-k
candidate lists are merged); ``DeviceEngine`` supplies the CUDA primitives.
torch is used only to allocate device buffers and to hand NCCL the n-length
partial products; all arithmetic is in the CUDA kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import check, lib
from .dist import LocalComm, merge_topk

_SCAL = 8  # device scalar slots: 0 loss, 1 mean(r), 2 sum(rt), 3 max|g|, 4 image sumsq


def _torch():
    import torch

    return torch


def torch_event():
    return _torch().cuda.Event(enable_timing=True)


class Genotypes:
    """What the engine needs to know about the genotype operand of a view.

    matrix  the (local shard of the) device-resident packed matrix
    rows    sample subset the view stands for (None = all), e.g. CV training rows
    u, v    device stats to standardise with (None = the handle's own)
    j_base  global index of local SNP 0;  p_global  SNPs over all shards
    comm    communicator joining the shards (LocalComm for one GPU)
    """

    def __init__(self, matrix, rows=None, u=None, v=None, j_base=0, p_global=None, comm=None):
        self.matrix = matrix
        self.handle = getattr(matrix, "handle", None)
        self.device = getattr(matrix, "device", None)
        self.n_full = matrix.n
        self.rows = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        self.u = u
        self.v = v
        self.j_base = int(j_base)
        self.p_local = matrix.p
        self.p_global = matrix.p if p_global is None else int(p_global)
        self.comm = comm if comm is not None else LocalComm()


class ShardEngine:
    """Sharded phases of the IHT loop over abstract per-shard primitives.

    Subclasses implement:
      _ax_partial(which, idx_l, w_l)   buffer `which` ("fit" | "img") = X_local[:, idx_l] w_l
      _buffer(which)                   the n-length buffer (handed to comm.allreduce_sum_)
      _finish_refresh(bcov, has_fit, sup_l) -> (loss, max|g_local|, g_cov, g[sup_l])
      _finish_image(wcov) -> sumsq
      _topk_local(mode, mu, k) -> (keys uint64, global idx, values) of the local top-k
      _scatter_beta(idx_l, vals), reset_beta(), gradient(), residuals()
    """

    def __init__(self, geno: Genotypes, c: int, kmax: int):
        self.geno = geno
        self.comm = geno.comm
        self.n = geno.n_full
        self.p = geno.p_local
        self.c = int(c)
        self.kmax = max(1, int(kmax))
        self.kernel_launches = 0

    # ------------------------------------------------------------- indexing
    def local_part(self, idx_global, w):
        """Entries of a global sparse vector owned by this shard (local indices)."""
        idx_global = np.asarray(idx_global, dtype=np.int64)
        w = np.asarray(w, dtype=np.float64)
        if self.comm.world == 1 and self.geno.j_base == 0:
            return idx_global, w
        lo, hi = self.geno.j_base, self.geno.j_base + self.p
        sel = (idx_global >= lo) & (idx_global < hi)
        return idx_global[sel] - lo, w[sel]

    def _assemble(self, idx_global, local_vals):
        """Values at a global index list whose entries are spread over shards."""
        if self.comm.world == 1:
            return np.asarray(local_vals, dtype=np.float64)
        idx_global = np.asarray(idx_global, dtype=np.int64)
        full = np.zeros(idx_global.size)
        lo, hi = self.geno.j_base, self.geno.j_base + self.p
        full[(idx_global >= lo) & (idx_global < hi)] = local_vals
        return self.comm.allreduce_sum_host(full)

    def _ax_global(self, which, idx_global, w):
        idx_l, w_l = self.local_part(idx_global, w)
        self._ax_partial(which, idx_l, w_l)
        if self.comm.world > 1:
            self.comm.allreduce_sum_(self._buffer(which))

    # --------------------------------------------------------------- phases
    def set_beta(self, old_idx, new_idx, new_w):
        """Dense per-shard beta: zero the old support, write the new one."""
        old_l, _ = self.local_part(old_idx, np.zeros(len(old_idx)))
        if old_l.size:
            self._scatter_beta(old_l, np.zeros(old_l.size))
        new_l, w_l = self.local_part(new_idx, new_w)
        if new_l.size:
            self._scatter_beta(new_l, w_l)

    def refresh(self, support, weights, bcov):
        """r, loss and the full gradient at (support, weights, bcov).

        Returns (loss, max|g_gen| over all shards, g_cov (c,), g on support)."""
        has_fit = len(support) > 0
        if has_fit:
            self._ax_global("fit", support, weights)
        sup_l, _ = self.local_part(support, np.zeros(len(support)))
        loss, gmax, gcov, g_loc = self._finish_refresh(bcov, has_fit, sup_l)
        if self.comm.world > 1:
            gmax = self.comm.allreduce_max(gmax)
        return loss, gmax, gcov, self._assemble(support, g_loc)

    def image_sumsq(self, idx, w, wcov) -> float:
        """|| X_idx w + C wcov ||^2 over the view's rows."""
        self._ax_global("img", idx, w)
        return self._finish_image(wcov)

    def topk(self, mode: int, mu: float, k: int):
        """Global top-k (sorted indices, values) of |g| (mode 0) or |beta - mu g| (mode 1)."""
        k_eff = min(int(k), self.kmax)
        keys, idx, vals = self._topk_local(mode, mu, k_eff)
        if self.comm.world > 1:
            # one all-gather of (key bits | index | value) per rank, 8 bytes each
            packed = np.zeros((3, k_eff), np.int64)
            packed[1] = -1
            packed[0, : keys.size] = keys.view(np.int64)
            packed[1, : idx.size] = idx
            packed[2, : vals.size] = np.asarray(vals, np.float64).view(np.int64)
            parts = self.comm.allgather_host(packed.reshape(-1))
            stacked = np.stack([p_.reshape(3, k_eff) for p_ in parts], axis=0)
            keys = stacked[:, 0].reshape(-1).view(np.uint64)
            idx = stacked[:, 1].reshape(-1)
            vals = np.ascontiguousarray(stacked[:, 2].reshape(-1)).view(np.float64)
        return merge_topk(keys, idx, vals, k_eff)


class DeviceEngine(ShardEngine):
    """CUDA primitives for ShardEngine on the shard's GPU."""

    def __init__(self, geno: Genotypes, y: np.ndarray, cov: np.ndarray | None, kmax: int):
        super().__init__(geno, 0 if cov is None else cov.shape[1], kmax)
        torch = _torch()
        _native.require_device(geno.device)
        self.torch = torch
        self.dev = torch.device("cuda", geno.device)
        self.h = geno.handle
        self.n_pad = int(lib().gi_padded_samples(self.h))
        f64, dev = torch.float64, self.dev
        with torch.cuda.device(self.dev):
            self.stream = torch.cuda.current_stream(self.dev)
        self.s = ctypes.c_void_p(self.stream.cuda_stream)

        y_full = np.zeros(self.n)
        keep = None
        if geno.rows is None:
            y_full[:] = y
            self.n_eff = float(self.n)
        else:
            y_full[geno.rows] = y
            keep = np.zeros(self.n, np.uint8)
            keep[geno.rows] = 1
            self.n_eff = float(geno.rows.size)
        self.y = torch.as_tensor(y_full, dtype=f64).to(dev)
        self.keep = None if keep is None else torch.as_tensor(keep).to(dev)
        if self.c:
            c_full = np.zeros((self.n, self.c))
            if geno.rows is None:
                c_full[:] = cov
            else:
                c_full[geno.rows] = cov
            self.C = torch.as_tensor(np.ascontiguousarray(c_full), dtype=f64).to(dev)
        else:
            self.C = None
        self.r = torch.zeros(self.n, dtype=f64, device=dev)
        self.bufs = {"fit": torch.zeros(self.n, dtype=f64, device=dev),
                     "img": torch.zeros(self.n, dtype=f64, device=dev)}
        self.rt = torch.zeros(self.n_pad, dtype=torch.float32, device=dev)
        self.g = torch.zeros(max(self.p, 1), dtype=f64, device=dev)
        self.beta = torch.zeros(max(self.p, 1), dtype=f64, device=dev)
        self.cvec = torch.zeros(max(self.c, 1) * 2, dtype=f64, device=dev)  # bcov | gcov
        self.scal = torch.zeros(_SCAL, dtype=f64, device=dev)
        self.partials = torch.zeros(int(lib().gi_red_partials()), dtype=f64, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        slots = int(lib().gi_topk_slots(max(self.p, 1), self.kmax))
        self.ckey = torch.zeros(slots, dtype=torch.int64, device=dev)
        self.cidx = torch.zeros(slots, dtype=torch.int64, device=dev)
        self.cval = torch.zeros(slots, dtype=f64, device=dev)
        self.oidx = torch.zeros(self.kmax, dtype=torch.int64, device=dev)
        self.oval = torch.zeros(self.kmax, dtype=f64, device=dev)
        self.okey = torch.zeros(self.kmax, dtype=torch.int64, device=dev)
        self.ocnt = torch.zeros(1, dtype=torch.int64, device=dev)
        self._kbuf = 0
        self._ensure_kbuf(max(2 * self.kmax, 64))
        # pinned staging for the small device->host traffic of each phase
        self.h_out = torch.zeros(_SCAL + 2 * self.c + 4 * self.kmax + 4, dtype=f64).pin_memory()
        self.u_ptr = None if geno.u is None else geno.u.data_ptr()
        self.v_ptr = None if geno.v is None else geno.v.data_ptr()
        self.aty_events = None  # list of (start, end) CUDA events when profiling
        # per-SNP (sum of dosages, observed count) over the view's rows: the fast
        # X^T r kernel restores the mean of r removed by centring with them
        self.s1cnt = None
        if geno.rows is not None:
            mask = np.zeros(self.n_pad // 16, np.uint32)
            np.bitwise_or.at(mask, geno.rows >> 4,
                             (1 << (2 * (geno.rows & 15))).astype(np.uint32))
            d_mask = torch.as_tensor(mask.view(np.int32)).to(dev)
            scratch = torch.zeros(2 * max(self.p, 1), dtype=f64, device=dev)
            self.s1cnt = torch.zeros(2 * max(self.p, 1), dtype=torch.int32, device=dev)
            P = _native.ptr
            check(lib().gi_dev_stats(self.h, P(d_mask), P(scratch), P(scratch) + 8 * self.p,
                                     P(self.s1cnt), self.s))
            self.kernel_launches += 1

    # ----------------------------------------------------- host<->device
    def _ensure_kbuf(self, k):
        if k <= self._kbuf:
            return
        torch = self.torch
        k = max(k, 2 * self._kbuf)
        self.d_idx = torch.zeros(k, dtype=torch.int64, device=self.dev)
        self.d_w = torch.zeros(k, dtype=torch.float64, device=self.dev)
        self._kbuf = k
        self._grow_pool(8 * k)

    def _grow_pool(self, words):
        """Pinned staging for H2D copies.  Every copy gets its own region (bump
        allocation) and regions are recycled only after a stream sync, so the host
        never overwrites bytes an enqueued copy has not read yet."""
        if getattr(self, "_pool_words", 0) >= words:
            return
        if getattr(self, "_pool_used", 0):
            self._sync()
        self._pool = self.torch.zeros(words, dtype=self.torch.float64).pin_memory()
        self._pool_words = words
        self._pool_used = 0

    def _stage(self, values: np.ndarray, kind: str):
        k = int(values.size)
        if self._pool_used + k > self._pool_words:
            self._sync()
            self._grow_pool(max(self._pool_words, 2 * k))
        lo = self._pool_used
        self._pool_used += k
        region = self._pool[lo:lo + k]
        if kind == "i64":
            region = region.view(self.torch.int64)
        region.numpy()[:] = values
        return region

    def _upload_sparse(self, idx_local, w) -> int:
        k = int(idx_local.size)
        if k == 0:
            return 0
        self._ensure_kbuf(k)
        self.d_idx[:k].copy_(self._stage(np.asarray(idx_local, np.int64), "i64"),
                             non_blocking=True)
        self.d_w[:k].copy_(self._stage(np.asarray(w, np.float64), "f64"), non_blocking=True)
        return k

    def _upload_cov(self, values) -> None:
        self.cvec[: self.c].copy_(self._stage(np.asarray(values, np.float64), "f64"),
                                  non_blocking=True)

    def _sync(self):
        self.stream.synchronize()
        self._pool_used = 0

    # -------------------------------------------------------- primitives
    def _buffer(self, which):
        return self.bufs[which]

    def _ax_partial(self, which, idx_l, w_l):
        P = _native.ptr
        k = self._upload_sparse(idx_l, w_l)
        check(lib().gi_dev_ax(self.h, self.u_ptr, self.v_ptr, P(self.d_idx), P(self.d_w), k,
                              P(self.bufs[which]), 0, self.s))
        self.kernel_launches += 1 if k else 0

    def _scatter_beta(self, idx_l, vals):
        P = _native.ptr
        k = self._upload_sparse(idx_l, vals)
        check(lib().gi_dev_scatter(k, P(self.d_idx), P(self.d_w), P(self.beta), self.s))
        self.kernel_launches += 1

    def reset_beta(self):
        self.beta.zero_()

    def _finish_refresh(self, bcov, has_fit, sup_l):
        P = _native.ptr
        L = lib()
        if self.c:
            self._upload_cov(bcov)
        cptr = P(self.cvec)
        gcov_ptr = cptr + 8 * self.c if self.c else None
        keep = P(self.keep) if self.keep is not None else None
        check(L.gi_dev_residual(self.n, P(self.y), P(self.bufs["fit"]) if has_fit else None,
                                P(self.C) if self.c else None, self.c, cptr if self.c else None,
                                keep, self.n_eff, P(self.r), P(self.scal), P(self.partials),
                                P(self.ticket), self.s))
        check(L.gi_dev_center(self.n, self.n_pad, P(self.r), keep, P(self.scal), P(self.rt),
                              P(self.partials), P(self.ticket), self.s))
        if self.p:
            ev = None
            if self.aty_events is not None:
                ev = (torch_event(), torch_event())
                ev[0].record(self.stream)
            check(L.gi_dev_aty_fast(self.h, self.u_ptr, self.v_ptr, P(self.s1cnt), P(self.rt),
                                    P(self.scal), -1.0, P(self.g), self.s))
            if ev is not None:
                ev[1].record(self.stream)
                self.aty_events.append(ev)
            check(L.gi_dev_maxabs(self.p, P(self.g), P(self.scal), 3, P(self.partials),
                                  P(self.ticket), self.s))
        if self.c:
            check(L.gi_dev_covgrad(self.n, P(self.C), self.c, P(self.r), gcov_ptr,
                                   P(self.partials), P(self.ticket), self.s))
        self.kernel_launches += 2 + (2 if self.p else 0) + (1 if self.c else 0)
        ks = int(sup_l.size)
        if ks:
            self._upload_sparse(sup_l, np.zeros(ks))
            check(L.gi_dev_gather(ks, P(self.d_idx), P(self.g), P(self.oval), self.s))
            self.kernel_launches += 1
        ho = self.h_out
        ho[:_SCAL].copy_(self.scal, non_blocking=True)
        if self.c:
            ho[_SCAL:_SCAL + self.c].copy_(self.cvec[self.c:2 * self.c], non_blocking=True)
        if ks:
            ho[_SCAL + self.c:_SCAL + self.c + ks].copy_(self.oval[:ks], non_blocking=True)
        self._sync()
        hv = ho.numpy()
        gmax = float(hv[3]) if self.p else 0.0
        return (float(hv[0]), gmax, hv[_SCAL:_SCAL + self.c].copy(),
                hv[_SCAL + self.c:_SCAL + self.c + ks].copy())

    def _finish_image(self, wcov) -> float:
        P = _native.ptr
        L = lib()
        img = self.bufs["img"]
        if wcov is not None and self.c:
            self._upload_cov(wcov)
            check(L.gi_dev_add_cov(self.n, P(self.C), self.c, P(self.cvec), P(img), self.s))
            self.kernel_launches += 1
        if self.keep is not None:
            img.mul_(self.keep)
        check(L.gi_dev_sumsq(self.n, P(img), P(self.scal), 4, P(self.partials), P(self.ticket),
                             self.s))
        self.kernel_launches += 1
        self.h_out[4:5].copy_(self.scal[4:5], non_blocking=True)
        self._sync()
        return float(self.h_out.numpy()[4])

    def _topk_local(self, mode, mu, k_eff):
        P = _native.ptr
        if self.p == 0 or k_eff <= 0:
            return np.zeros(0, np.uint64), np.zeros(0, np.int64), np.zeros(0)
        check(lib().gi_dev_topk(self.p, k_eff, mode, P(self.beta), P(self.g), float(mu),
                                self.geno.j_base, P(self.ckey), P(self.cidx), P(self.cval),
                                P(self.oidx), P(self.oval), P(self.okey), P(self.ocnt), self.s))
        self.kernel_launches += 2
        f64 = self.torch.float64
        ho = self.h_out
        base = _SCAL + 2 * self.c
        ho[base:base + k_eff].copy_(self.oidx[:k_eff].view(f64), non_blocking=True)
        ho[base + k_eff:base + 2 * k_eff].copy_(self.oval[:k_eff], non_blocking=True)
        ho[base + 2 * k_eff:base + 3 * k_eff].copy_(self.okey[:k_eff].view(f64), non_blocking=True)
        ho[base + 3 * k_eff:base + 3 * k_eff + 1].copy_(self.ocnt.view(f64), non_blocking=True)
        self._sync()
        hv = ho.numpy()
        cnt = int(hv[base + 3 * k_eff:base + 3 * k_eff + 1].view(np.int64)[0])
        idx = hv[base:base + cnt].view(np.int64).copy()
        vals = hv[base + k_eff:base + k_eff + cnt].copy()
        keys = hv[base + 2 * k_eff:base + 2 * k_eff + cnt].view(np.uint64).copy()
        return keys, idx, vals

    def gradient(self) -> np.ndarray:
        """Local genetic gradient (host copy)."""
        return self.g[: self.p].cpu().numpy().copy()

    def residuals(self) -> np.ndarray:
        r = self.r.cpu().numpy()
        return r if self.geno.rows is None else r[self.geno.rows].copy()
