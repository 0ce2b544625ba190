"""Multi-GPU driver: one process per GPU, rows of every mode sharded across the
ranks by contiguous nnz-balanced ranges.

Each rank builds a shard context (`vest_ctx_create_shard`) over the full
tensor that updates and traverses only its own rows, and installs
communication hooks (`vest_ctx_set_comm`) that the library calls at the exchange
points of the CD sweep:

* allgather_rows(mode, buf, ld): after each factor mode (and for the factor
  responsibility tables) every rank broadcasts its rows [lo_r, hi_r) of the
  row-major buffer -- one NCCL broadcast per rank over NVLink/NVSwitch;
* allreduce_sum(p, n): core block statistics [T | C], sum of squared
  residuals, core-responsibility statistics -- an NCCL all-reduce.

Everything else (block solves, prune selection, sparsity) then runs
identically on every rank on identical data, so the replicas stay consistent.

`NcclNative` (the production path, bench.py under torchrun) installs a native
NCCL communicator in the library (vest_ctx_set_nccl): the collectives are
issued by the library on its own stream, no Python per exchange.  `TorchComm`
implements the hooks as host callbacks with torch.distributed (NCCL for device
pointers, gloo for host pointers in the CPU tests); `LocalGroup` emulates W
ranks as W threads of one process on one GPU (host-synchronised exchanges,
no device-side waits) for single-GPU testing of the sharded path.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, f64p, ptr, u32p, u64p
from .sparsetuck import Device, SparseTensor

ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_uint64, C.c_void_p)
ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_uint64, C.c_void_p)


class VestComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum", ALLREDUCE), ("allgather_rows", ALLGATHER)]


def partition(x: SparseTensor, world: int, row_cost: Optional[int] = None):
    """Per-mode row bounds [world + 1] balanced by work: observed entries plus
    `row_cost` entry-equivalents per non-empty row (the per-row solve and the
    short-row kernel's one-lane-per-row cost; VEST_ROW_COST overrides), through
    vest_partition_rows over the weights' prefix sums."""
    import os
    if row_cost is None:
        row_cost = int(os.environ.get("VEST_ROW_COST", "8"))
    L = _lib.lib()
    bounds = []
    for n in range(x.order()):
        counts = np.bincount(np.asarray(x.coords[:, n], np.int64), minlength=int(x.dims[n]))
        if row_cost:
            counts = counts + row_cost * (counts > 0)
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
        b = np.zeros(world + 1, np.uint64)
        check(L.vest_partition_rows(ptr(off, u64p), int(x.dims[n]), world, ptr(b, u64p)))
        bounds.append(b)
    return bounds


class ShardDevice(Device):
    """A Device that owns rank `rank`'s rows and exchanges through `comm`."""

    def __init__(self, x: SparseTensor, ranks: Sequence[int], rank: int, world: int, comm, device: int = 0,
                 bounds=None):
        self.bounds = bounds if bounds is not None else partition(x, world)
        self.rank, self.world = rank, world
        lo = np.asarray([int(b[rank]) for b in self.bounds], np.uint64)
        hi = np.asarray([int(b[rank + 1]) for b in self.bounds], np.uint64)
        self.x = x
        self.dims = [int(d) for d in x.dims]
        self.ranks = [int(r) for r in ranks]
        self.order = len(self.dims)
        L = _lib.lib()
        self._L = L
        d = np.asarray(self.dims, np.uint64)
        r = np.asarray(self.ranks, np.uint64)
        coords = np.ascontiguousarray(x.coords, np.uint32).reshape(-1)
        vals = np.ascontiguousarray(x.values, np.float64)
        h = C.c_void_p()
        check(L.vest_ctx_create_shard(self.order, ptr(d, u64p), x.nnz(), ptr(coords, u32p), ptr(vals, f64p),
                                      ptr(r, u64p), device, ptr(lo, u64p), ptr(hi, u64p), C.byref(h)))
        self.h = h
        self.comm = comm
        if isinstance(comm, NcclNative):
            comm.install(self)
        else:
            self._hooks = comm.hooks(self)  # keep the ctypes callbacks alive
            check(L.vest_ctx_set_comm(self.h, C.cast(C.pointer(self._hooks), C.c_void_p)))

    def local_nnz(self, mode: int) -> int:
        return int(self._L.vest_ctx_local_nnz(self.h, mode))


# ----------------------------------------------------------- native NCCL --
class NcclNative:
    """The exchanges as native NCCL collectives on the library's stream
    (vest_ctx_set_nccl): rank 0 makes the unique id, torch.distributed
    distributes it (any backend), every rank installs the communicator with the
    row bounds of every mode.  No host callback per exchange."""

    def install(self, dev: "ShardDevice"):
        import torch.distributed as dist

        L = _lib.lib()
        buf = (C.c_char * 128)()
        if dev.rank == 0:
            check(L.vest_nccl_unique_id(C.cast(buf, C.c_void_p)))
        obj = [bytes(buf) if dev.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        bounds = np.concatenate([np.asarray(b, np.uint64) for b in dev.bounds])
        check(L.vest_ctx_set_nccl(dev.h, dev.rank, dev.world, C.cast(uid, C.c_void_p), ptr(bounds, u64p)))


# ------------------------------------------------------------- torch comm --
class TorchComm:
    """Hooks over torch.distributed.  Device pointers (NCCL) are wrapped as
    torch tensors through __cuda_array_interface__ and the collectives are
    issued on the library's stream; host pointers (gloo) are wrapped through
    numpy."""

    def __init__(self, device: str = "cuda"):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.device = device

    def _wrap(self, p, n):
        torch = self.torch
        if self.device == "cpu":
            arr = np.ctypeslib.as_array(p, shape=(int(n),))
            return torch.from_numpy(arr)

        class _Cai:
            __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                        "data": (C.cast(p, C.c_void_p).value, False), "version": 3}

        return torch.as_tensor(_Cai(), device="cuda")

    def _stream_ctx(self, stream):
        torch = self.torch
        if self.device == "cpu" or not stream:
            import contextlib
            return contextlib.nullcontext()
        return torch.cuda.stream(torch.cuda.ExternalStream(stream))

    def allreduce(self, p, n, stream):
        t = self._wrap(p, n)
        with self._stream_ctx(stream):
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return 0

    def allgather_rows(self, dev: "ShardDevice", mode, base, ld, stream):
        b = dev.bounds[mode]
        n = int(b[-1]) * int(ld)
        t = self._wrap(base, n)
        with self._stream_ctx(stream):
            for r in range(dev.world):
                lo, hi = int(b[r]) * int(ld), int(b[r + 1]) * int(ld)
                if hi > lo:
                    self.dist.broadcast(t[lo:hi], src=r)
        return 0

    def hooks(self, dev: "ShardDevice") -> VestComm:
        def ar(user, p, n, stream):
            try:
                return self.allreduce(p, n, stream)
            except Exception:  # noqa: BLE001 -- reported to the library as a failed hook
                return 1

        def ag(user, mode, base, ld, stream):
            try:
                return self.allgather_rows(dev, mode, base, ld, stream)
            except Exception:  # noqa: BLE001
                return 1

        return VestComm(None, ALLREDUCE(ar), ALLGATHER(ag))


# ------------------------------------------------ timing-only null exchange --
class NullComm:
    """Hooks that exchange nothing: one rank's shard context runs its own share
    of the sweep alone (bench.py --shard-emulate W, per-GPU device time at W
    GPUs).  Results are NOT the sharded model's (nothing is summed/gathered);
    the device work per iteration is the rank's -- timing only."""

    def hooks(self, dev: "ShardDevice") -> VestComm:
        def ar(user, p, n, stream):
            return 0

        def ag(user, mode, base, ld, stream):
            return 0

        return VestComm(None, ALLREDUCE(ar), ALLGATHER(ag))


# --------------------------------------------------- one-GPU emulated group --
class LocalGroup:
    """W shard contexts of one process on one GPU, driven by W threads.  Each
    exchange: every thread synchronises its own stream and waits at a barrier;
    thread 0 performs the sum / row copy on the device (torch, default stream,
    then device-synchronised); a second barrier releases the threads.  No kernel
    ever waits on another, so this is safe on a single GPU."""

    def __init__(self, world: int):
        import torch

        self.torch = torch
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: list = [None] * world
        self.error: Optional[BaseException] = None

    def _tensor(self, p, n):
        torch = self.torch

        class _Cai:
            __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                        "data": (C.cast(p, C.c_void_p).value, False), "version": 3}

        return torch.as_tensor(_Cai(), device="cuda")

    def _exchange(self, rank, stream, payload, fn):
        torch = self.torch
        torch.cuda.synchronize()
        self.slots[rank] = payload
        self.barrier.wait()
        if rank == 0:
            try:
                fn(self.slots)
                torch.cuda.synchronize()
            except BaseException as e:  # noqa: BLE001
                self.error = e
        self.barrier.wait()
        return 1 if self.error else 0

    def hooks_for(self, rank: int):
        group = self

        class _Comm:
            def hooks(self, dev):
                def ar(user, p, n, stream):
                    def fn(slots):
                        ts = [group._tensor(q, m) for (q, m) in slots]
                        s = ts[0].clone()
                        for t in ts[1:]:
                            s += t
                        for t in ts:
                            t.copy_(s)
                    return group._exchange(rank, stream, (p, n), fn)

                def ag(user, mode, base, ld, stream):
                    b = dev.bounds[mode]
                    n = int(b[-1]) * int(ld)

                    def fn(slots):
                        ts = [group._tensor(q, n) for (q, _) in slots]
                        for r in range(group.world):
                            lo, hi = int(b[r]) * int(ld), int(b[r + 1]) * int(ld)
                            for q, t in enumerate(ts):
                                if q != r and hi > lo:
                                    t[lo:hi].copy_(ts[r][lo:hi])
                    return group._exchange(rank, stream, (base, n), fn)

                return VestComm(None, ALLREDUCE(ar), ALLGATHER(ag))

        return _Comm()

    def run(self, fns):
        """Run fns[r]() on W threads (one per emulated rank); returns results."""
        out = [None] * self.world
        errs = [None] * self.world

        def body(r):
            try:
                out[r] = fns[r]()
            except BaseException as e:  # noqa: BLE001
                errs[r] = e
                try:
                    self.barrier.abort()
                except Exception:
                    pass

        th = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        return out
