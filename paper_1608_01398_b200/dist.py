"""SNP-block sharding across GPUs (one process per GPU, torch.distributed).

The genotype matrix is split into contiguous SNP blocks, one per rank
(SURVEY.md section 8(e)).  Every rank runs the same IHT control flow on
identical reduced values, so all ranks take identical branches.  The only data
exchanged per iteration are n-length partial products (X_S w summed across
shards: NCCL all-reduce on device buffers) and the k-candidate top-k lists
(all-gather), plus a few scalars.

``LocalComm`` is the single-process communicator; ``TorchComm`` wraps the
default torch.distributed process group (NCCL across GPUs; gloo for the CPU
tests).
"""

from __future__ import annotations

import traceback

import numpy as np


def shard_range(p: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous SNP block [j0, j1) of ``rank``; blocks differ by at most one SNP."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world size / rank")
    base, extra = divmod(int(p), int(world))
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)


class LocalComm:
    world = 1
    rank = 0

    def allreduce_sum_(self, tensor):
        return tensor

    def allreduce_max(self, value: float) -> float:
        return float(value)

    def allreduce_sum_host(self, array: np.ndarray) -> np.ndarray:
        return np.asarray(array, dtype=np.float64)

    def allgather_host(self, array: np.ndarray) -> list:
        return [np.asarray(array)]

    def allreduce_host(self, array: np.ndarray, op: str) -> np.ndarray:
        return np.asarray(array, dtype=np.float64)


class TorchComm:
    """Collectives on the default process group.  Device buffers go straight to
    NCCL; with the gloo backend (CPU tests) CUDA buffers are staged on the host."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)

    def _device(self):
        import torch

        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def allreduce_sum_(self, tensor):
        if self.backend != "nccl" and tensor.is_cuda:
            host = tensor.cpu()
            self.dist.all_reduce(host, group=self.group)
            tensor.copy_(host)
        else:
            self.dist.all_reduce(tensor, group=self.group)
        return tensor

    def allreduce_max(self, value: float) -> float:
        import torch

        t = torch.tensor([float(value)], dtype=torch.float64, device=self._device())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allreduce_sum_host(self, array: np.ndarray) -> np.ndarray:
        import torch

        t = torch.as_tensor(np.asarray(array, dtype=np.float64)).to(self._device())
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def allgather_host(self, array: np.ndarray) -> list:
        import torch

        t = torch.as_tensor(np.ascontiguousarray(array)).to(self._device())
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def allreduce_host(self, array: np.ndarray, op: str) -> np.ndarray:
        import torch

        t = torch.as_tensor(np.asarray(array, dtype=np.float64)).to(self._device())
        red = self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX
        self.dist.all_reduce(t, op=red, group=self.group)
        return t.cpu().numpy()


class NativeComm:
    """A gi_comm* for the native sharded loop (gi_fit_sharded).

    With the NCCL backend the library runs its own NCCL communicator (rank 0's
    unique id is broadcast over the torch process group) and reduces device
    buffers in place on the fit's stream.  Otherwise (gloo: several ranks may
    share one GPU) the library calls back into ``comm``'s host collectives."""

    def __init__(self, comm, device: int):
        import ctypes

        from . import _native

        self.comm = comm
        self.raw = ctypes.c_void_p(0)
        L = _native.lib()
        use_nccl = getattr(comm, "backend", None) == "nccl" and L.gi_comm_nccl_available()
        if use_nccl:
            uid = (ctypes.c_uint8 * 128)()
            if comm.rank == 0:
                _native.check(L.gi_comm_nccl_unique_id(uid))
            box = [bytes(uid)]
            comm.dist.broadcast_object_list(box, src=0, group=comm.group)
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
            _native.check(L.gi_comm_create_nccl(uid, comm.world, comm.rank, device,
                                                ctypes.byref(self.raw)))
            self.kind = "nccl"
        else:
            def allreduce(_ctx, buf, count, op):
                try:
                    arr = np.ctypeslib.as_array(buf, shape=(count,))
                    arr[:] = comm.allreduce_host(arr.copy(), "sum" if op == 0 else "max")
                    return 0
                except Exception:  # reported by the library as a failed collective
                    traceback.print_exc()
                    return -1

            def allgather(_ctx, send, count, recv):
                try:
                    src = np.ctypeslib.as_array(send, shape=(count,)).copy()
                    dst = np.ctypeslib.as_array(recv, shape=(count * comm.world,))
                    dst[:] = np.concatenate(comm.allgather_host(src))
                    return 0
                except Exception:
                    traceback.print_exc()
                    return -1

            # keep the ctypes thunks alive as long as the communicator
            self._ar = _native.ALLREDUCE_FN(allreduce)
            self._ag = _native.ALLGATHER_FN(allgather)
            _native.check(L.gi_comm_create_callbacks(comm.world, comm.rank, None, self._ar,
                                                     self._ag, ctypes.byref(self.raw)))
            self.kind = "callbacks"

    def __del__(self):
        try:
            from . import _native

            if self.raw:
                _native.lib().gi_comm_free(self.raw)
                self.raw = None
        except Exception:
            pass


def merge_topk(keys: np.ndarray, idx: np.ndarray, vals: np.ndarray, k: int):
    """Global top-k from per-shard candidate lists under (|value| desc, index asc).

    ``keys`` are the uint64 bit patterns of |value| plus one (0 = empty slot),
    exactly as gi_dev_topk emits them; each shard's list is already its exact
    local top-k under the same order, so their union contains the global one.
    Returns indices sorted ascending and the matching values.
    """
    keys = np.asarray(keys, dtype=np.uint64)
    live = keys != 0
    keys, idx, vals = keys[live], np.asarray(idx)[live], np.asarray(vals)[live]
    order = np.lexsort((idx, ~keys))  # key descending, then index ascending
    take = order[:k]
    sel = np.argsort(idx[take], kind="stable")
    return idx[take][sel].astype(np.int64), vals[take][sel]


class ShardedGenotypes:
    """This rank's SNP block of a matrix sharded over ``comm.world`` GPUs.

    Behaves like a packed matrix of the GLOBAL shape for the solver (global
    SNP indices everywhere); the fit engine runs on the local block and joins
    the shards through ``comm``."""

    def __init__(self, local, j_base: int, p_global: int, comm):
        self.local = local
        self.j_base = int(j_base)
        self.p = int(p_global)
        self.n = local.n
        self.device = local.device
        self.comm = comm

    @classmethod
    def synthetic(cls, n: int, p: int, seed: int, comm, device: int, maf_range=(0.05, 0.5),
                  missing_rate: float = 0.0):
        from .geno_matrix import PackedGenotypeMatrix

        j0, j1 = shard_range(p, comm.world, comm.rank)
        local = PackedGenotypeMatrix.synthetic(n, j1 - j0, seed, maf_range=maf_range,
                                               missing_rate=missing_rate, device=device,
                                               j_base=j0)
        return cls(local, j0, p, comm)

    def engine_genotypes(self):
        from .engine import Genotypes

        return Genotypes(self.local, j_base=self.j_base, p_global=self.p, comm=self.comm)

    def native_comm(self) -> "NativeComm":
        """The library-side communicator (created once per process group)."""
        cached = getattr(self.comm, "_native_comm", None)
        if cached is None:
            cached = NativeComm(self.comm, self.device)
            self.comm._native_comm = cached
        return cached

    def ax_columns(self, idx, w) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.int64)
        w = np.asarray(w, dtype=np.float64)
        if idx.size and (idx.min() < 0 or idx.max() >= self.p):
            raise IndexError("variant index out of range")
        sel = (idx >= self.j_base) & (idx < self.j_base + self.local.p)
        part = self.local.ax_columns(idx[sel] - self.j_base, w[sel])
        return self.comm.allreduce_sum_host(part)
