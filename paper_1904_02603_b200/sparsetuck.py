"""Python mirror of the reference's sparsetuck:: API on the B200 path.

Every name, argument and error here follows /root/reference/proj/include/
sparsetuck/*.hpp (cited per function) so code written against the reference
library ports one-to-one.  Two layers:

* `Device` -- the fast path: one device context (libvest_cuda.so, include/vest.h)
  holds the tensor's per-mode CSF and the model in HBM; methods run the hot
  path without host round trips.  `fit()` drives it.
* module functions (`update_all_factors(m, x, idx, ...)` etc.) -- the drop-in
  slow path with the reference's signatures: the host `TuckerModel` is synced
  to the device context cached on the tensor, the kernel runs, and the result is
  copied back into the caller's model (the reference mutates in place).

There is no CPU fallback: all numerics run in the CUDA kernels; this module
only validates arguments, moves buffers and runs the host-side control
(PruneSchedule / StopController), like the reference's trainer.hpp.
"""
from __future__ import annotations

import ctypes as C
import enum
import hashlib
import math
import os
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, f64p, ptr, u8p, u32p, u64p


class Regularizer(enum.IntEnum):  # updates.hpp:15
    LF = 0
    L1 = 1


class StopMode(enum.IntEnum):  # pruning.hpp:35
    Manual = 0
    Auto = 1


# --------------------------------------------------------------------- tensor --
@dataclass
class SparseTensor:
    """COO observed entries (sparse_tensor.hpp:29-50)."""

    dims: list
    coords: np.ndarray  # (nnz, order) uint32, entry-major
    values: np.ndarray  # (nnz,) float64
    _devices: dict = field(default_factory=dict, repr=False, compare=False)

    def order(self) -> int:
        return len(self.dims)

    def nnz(self) -> int:
        return int(self.values.shape[0])

    def entry(self, e: int) -> np.ndarray:
        return self.coords[e]

    def frobenius_norm(self) -> float:
        # serial sum in entry order (sparse_tensor.hpp:45-49)
        acc = 0.0
        for v in self.values.tolist():
            acc += v * v
        return math.sqrt(acc)


def make_tensor(dims: Sequence[int], coords, values) -> SparseTensor:
    """make_tensor / check_tensor (sparse_tensor.hpp:68-105)."""
    dims = [int(d) for d in dims]
    n = len(dims)
    if n == 0:
        raise ValueError("tensor order must be at least 1")
    if any(d == 0 for d in dims):
        raise ValueError("tensor dimensions must be positive")
    values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    coords = np.ascontiguousarray(coords, dtype=np.uint32)
    if coords.size != values.size * n:
        raise ValueError("coordinate buffer size does not match nnz * order")
    coords = coords.reshape(values.size, n)
    if values.size and (coords >= np.asarray(dims, dtype=np.uint64)[None, :]).any():
        raise ValueError("coordinate out of bounds")
    if values.size > 1:
        order = np.lexsort(coords.T[::-1])
        srt = coords[order]
        if (srt[1:] == srt[:-1]).all(axis=1).any():
            raise ValueError("duplicate coordinate in tensor")
    return SparseTensor(dims, coords, values)


# ---------------------------------------------------------------- data formats --
def _coo_from_handle(h) -> SparseTensor:
    L = _lib.lib()
    try:
        order, nnz = C.c_int(), C.c_uint64()
        _lib.io_check(L.vest_coo_info(h, C.byref(order), C.byref(nnz), None, None, None))
        dims = np.zeros(order.value, np.uint64)
        cp, vp_ = u32p(), f64p()
        _lib.io_check(L.vest_coo_info(h, None, None, ptr(dims, u64p), C.byref(cp), C.byref(vp_)))
        n, k = int(nnz.value), int(order.value)
        coords = np.ctypeslib.as_array(cp, shape=(max(n * k, 1),))[: n * k].copy().reshape(n, k) if n else \
            np.zeros((0, k), np.uint32)
        values = np.ctypeslib.as_array(vp_, shape=(max(n, 1),))[:n].copy() if n else np.zeros(0)
        return SparseTensor([int(d) for d in dims], coords, values)
    finally:
        L.vest_coo_free(h)


def load_coo(path, one_based: bool = False, threads: int = 0) -> SparseTensor:
    """load_coo (sparse_tensor.hpp:139-209): parallel parse, the reference's
    rules and messages, then make_tensor's validation."""
    h = C.c_void_p()
    _lib.io_check(_lib.lib().vest_coo_load(str(path).encode(), int(one_based), int(threads), C.byref(h)))
    return _coo_from_handle(h)


def save_coo(x: SparseTensor, path) -> None:
    """save_coo (sparse_tensor.hpp:211-228): byte-identical text."""
    d = np.asarray(x.dims, np.uint64)
    c = np.ascontiguousarray(x.coords, np.uint32).reshape(-1)
    v = np.ascontiguousarray(x.values, np.float64)
    _lib.io_check(_lib.lib().vest_coo_save(str(path).encode(), x.order(), ptr(d, u64p), x.nnz(),
                                           ptr(c, u32p), ptr(v, f64p)))


def save_coo_cache(x: SparseTensor, path) -> None:
    """Binary tensor cache (vest_coo_cache_save): parse a large input once."""
    d = np.asarray(x.dims, np.uint64)
    c = np.ascontiguousarray(x.coords, np.uint32).reshape(-1)
    v = np.ascontiguousarray(x.values, np.float64)
    _lib.io_check(_lib.lib().vest_coo_cache_save(str(path).encode(), x.order(), ptr(d, u64p), x.nnz(),
                                                 ptr(c, u32p), ptr(v, f64p)))


def load_coo_cache(path) -> SparseTensor:
    h = C.c_void_p()
    _lib.io_check(_lib.lib().vest_coo_cache_load(str(path).encode(), C.byref(h)))
    return _coo_from_handle(h)


@dataclass
class ModeIndex:
    """Per-mode CSR (sparse_tensor.hpp:109-117): read back from the device CSF."""

    offsets: list
    ids: list

    def slice(self, mode: int, i: int) -> np.ndarray:
        off = self.offsets[mode]
        return self.ids[mode][int(off[i]):int(off[i + 1])]


def build_mode_index(x: SparseTensor) -> ModeIndex:
    """build_mode_index (sparse_tensor.hpp:119-137), built on the device."""
    dev = _tensor_device(x, [1] * x.order())
    off, ids = [], []
    for n in range(x.order()):
        o, i = dev.mode_index(n)
        off.append(o)
        ids.append(i)
    return ModeIndex(off, ids)


# ---------------------------------------------------------------------- model --
@dataclass
class TuckerModel:
    """Dense core + factor matrices with pruning masks (tucker_model.hpp:21-47)."""

    dims: list
    ranks: list
    core: np.ndarray
    core_mask: np.ndarray
    factors: list
    factor_masks: list

    def order(self) -> int:
        return len(self.dims)

    def core_size(self) -> int:
        return int(np.prod(self.ranks))

    def factor_at(self, n: int, i: int, j: int) -> float:
        return float(self.factors[n][i, j])

    def num_elements(self) -> int:
        return self.core_size() + sum(int(d) * int(r) for d, r in zip(self.dims, self.ranks))

    def copy(self) -> "TuckerModel":
        return TuckerModel(list(self.dims), list(self.ranks), self.core.copy(), self.core_mask.copy(),
                           [f.copy() for f in self.factors], [m.copy() for m in self.factor_masks])


def _zero_model(dims, ranks) -> TuckerModel:
    g = int(np.prod(ranks))
    return TuckerModel(list(dims), list(ranks), np.zeros(g), np.zeros(g, np.uint8),
                       [np.zeros((int(d), int(r))) for d, r in zip(dims, ranks)],
                       [np.zeros((int(d), int(r)), np.uint8) for d, r in zip(dims, ranks)])


def init_random(dims: Sequence[int], ranks: Sequence[int], seed: int) -> TuckerModel:
    """init_random (tucker_model.hpp:88-108): identical draws to the reference."""
    if len(dims) != len(ranks):
        raise ValueError("ranks/dims order mismatch")
    m = _zero_model(dims, ranks)
    d = np.asarray(dims, np.uint64)
    r = np.asarray(ranks, np.uint64)
    fp = (f64p * len(dims))(*[ptr(f, f64p) for f in m.factors])
    check(_lib.lib().vest_init_random_host(len(dims), ptr(d, u64p), ptr(r, u64p), seed, ptr(m.core, f64p), fp))
    return m


@dataclass
class Residuals:  # tucker_model.hpp:161-166
    r: Optional[np.ndarray]
    sum_sq: float = 0.0
    x_norm: float = 0.0
    re: float = 0.0


@dataclass
class ResponsibilityTable:  # pruning.hpp:88-91
    core: np.ndarray
    factors: list
    base_re: float = 0.0


@dataclass
class PruneCounts:  # pruning.hpp:193-203
    core: int = 0
    factors: list = field(default_factory=list)

    def total(self) -> int:
        return self.core + sum(self.factors)


# --------------------------------------------------------------------- device --
class Device:
    """A device context: the tensor's CSF per mode + one model, resident in HBM."""

    def __init__(self, x: SparseTensor, ranks: Sequence[int], device: int = 0):
        self.x = x
        self.dims = [int(d) for d in x.dims]
        self.ranks = [int(r) for r in ranks]
        self.order = len(self.dims)
        if len(self.ranks) != self.order:
            raise ValueError("ranks order mismatch")
        L = _lib.lib()
        self._L = L
        d = np.asarray(self.dims, np.uint64)
        r = np.asarray(self.ranks, np.uint64)
        coords = np.ascontiguousarray(x.coords, np.uint32).reshape(-1)
        vals = np.ascontiguousarray(x.values, np.float64)
        h = C.c_void_p()
        check(L.vest_ctx_create(self.order, ptr(d, u64p), x.nnz(), ptr(coords, u32p), ptr(vals, f64p),
                                ptr(r, u64p), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self._L.vest_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- context
    def stream(self) -> int:
        return self._L.vest_ctx_stream(self.h) or 0

    def device_bytes(self) -> int:
        return int(self._L.vest_ctx_device_bytes(self.h))

    def specialised(self) -> bool:
        return bool(self._L.vest_ctx_specialised(self.h))

    def force_generic(self, on: bool = True):
        check(self._L.vest_ctx_force_generic(self.h, 1 if on else 0))

    def set_sparse_delta(self, mode: int):
        """Mask-specialised delta contraction: -1 auto, 0 off, 1 on."""
        check(self._L.vest_ctx_set_sparse_delta(self.h, int(mode)))

    def set_sparse_fused(self, mode: int):
        """-1 auto (= 0), 0: mask-specialised delta through HBM + statistics
        kernel, 1: one fused kernel per factor mode (bit-identical, slower)."""
        check(self._L.vest_ctx_set_sparse_fused(self.h, int(mode)))

    def set_gather_f32(self, on: bool):
        """fp32 mode of the generated (NVRTC) kernels: fp32 copies of the gathered
        factor rows, fp32 contraction of delta and of the core passes' fiber
        products; every Gram, solve, residual, the factors and the core stay
        fp64.  For fp32 workloads (BASELINE config 4)."""
        check(self._L.vest_ctx_set_gather_f32(self.h, 1 if on else 0))

    def set_core_gen(self, mode: int):
        """Plan-specialised core-sweep passes: -1 auto, 0 off, 1 on."""
        check(self._L.vest_ctx_set_core_gen(self.h, int(mode)))

    def sparse_delta_active(self) -> bool:
        return bool(self._L.vest_ctx_sparse_delta_active(self.h))

    def set_core_block(self, fibers: int):
        check(self._L.vest_ctx_set_core_block(self.h, fibers))

    def mode_index(self, mode: int):
        off = np.zeros(self.dims[mode] + 1, np.uint64)
        ids = np.zeros(max(self.x.nnz(), 1), np.uint32)
        check(self._L.vest_get_mode_index(self.h, mode, ptr(off, u64p), ptr(ids, u32p)))
        return off, ids[: self.x.nnz()]

    # -- model
    def init_random(self, seed: int):
        check(self._L.vest_init_random(self.h, seed))

    def set_model(self, m: TuckerModel):
        if list(m.dims) != self.dims or list(m.ranks) != self.ranks:
            raise ValueError("model/tensor shape mismatch")
        core = np.ascontiguousarray(m.core, np.float64)
        cm = np.ascontiguousarray(m.core_mask, np.uint8)
        fs = [np.ascontiguousarray(f, np.float64) for f in m.factors]
        ms = [np.ascontiguousarray(k, np.uint8) for k in m.factor_masks]
        fp = (f64p * self.order)(*[ptr(f, f64p) for f in fs])
        mp = (u8p * self.order)(*[ptr(k, u8p) for k in ms])
        check(self._L.vest_set_model(self.h, ptr(core, f64p), ptr(cm, u8p), fp, mp))

    def get_model(self, into: Optional[TuckerModel] = None) -> TuckerModel:
        m = into if into is not None else _zero_model(self.dims, self.ranks)
        fp = (f64p * self.order)(*[ptr(f, f64p) for f in m.factors])
        mp = (u8p * self.order)(*[ptr(k, u8p) for k in m.factor_masks])
        check(self._L.vest_get_model(self.h, ptr(m.core, f64p), ptr(m.core_mask, u8p), fp, mp))
        return m

    # -- hot path
    def update_all_factors(self, reg: int, lam: float):
        check(self._L.vest_update_all_factors(self.h, int(reg), float(lam)))

    def update_factor_mode(self, mode: int, reg: int, lam: float):
        check(self._L.vest_update_factor_mode(self.h, mode, int(reg), float(lam)))

    def update_factor_row(self, reg: int, mode: int, row: int, lam: float):
        check(self._L.vest_update_factor_row(self.h, int(reg), mode, row, float(lam)))

    def update_core(self, reg: int, lam: float):
        check(self._L.vest_update_core(self.h, int(reg), float(lam)))

    def compute_residuals(self, want_r: bool = False) -> Residuals:
        r = np.zeros(max(self.x.nnz(), 1)) if want_r else None
        ss, xn, re = C.c_double(), C.c_double(), C.c_double()
        check(self._L.vest_compute_residuals(self.h, ptr(r, f64p) if want_r else None, C.byref(ss),
                                             C.byref(xn), C.byref(re)))
        return Residuals(r[: self.x.nnz()] if want_r else None, ss.value, xn.value, re.value)

    def cd_iteration(self, reg: int, lam: float) -> float:
        re = C.c_double()
        check(self._L.vest_cd_iteration(self.h, int(reg), float(lam), C.byref(re)))
        return re.value

    def cd_iteration_host(self, m: TuckerModel, reg: int, lam: float) -> float:
        """One CD iteration on a host model, updated in place (vest_cd_iteration_host:
        upload, iterate, factors streamed back as each mode finishes)."""
        if list(m.dims) != self.dims or list(m.ranks) != self.ranks:
            raise ValueError("model/tensor shape mismatch")
        for a, dt in [(m.core, np.float64), (m.core_mask, np.uint8)] + [(f, np.float64) for f in m.factors] + \
                [(k, np.uint8) for k in m.factor_masks]:
            if a.dtype != dt or not a.flags.c_contiguous or not a.flags.writeable:
                raise ValueError("host model arrays must be writeable C-contiguous float64/uint8")
        fp = (f64p * self.order)(*[ptr(f, f64p) for f in m.factors])
        mp = (u8p * self.order)(*[ptr(k, u8p) for k in m.factor_masks])
        re = C.c_double()
        check(self._L.vest_cd_iteration_host(self.h, ptr(m.core, f64p), ptr(m.core_mask, u8p), fp, mp, int(reg),
                                              float(lam), C.byref(re)))
        return re.value

    def compute_delta(self, at, mode: int) -> np.ndarray:
        a = np.ascontiguousarray(at, np.uint32).reshape(-1)
        out = np.zeros(self.ranks[mode])
        check(self._L.vest_compute_delta(self.h, ptr(a, u32p), mode, ptr(out, f64p)))
        return out

    def row_stats(self, mode: int, row: int):
        """compute_row_stats (updates.hpp:64-79), bit-identical: (delta of the
        slice's last entry, gram J x J, xdelta)."""
        J = self.ranks[mode]
        d, g, x = np.zeros(J), np.zeros(J * J), np.zeros(J)
        check(self._L.vest_compute_row_stats(self.h, mode, row, ptr(g, f64p), ptr(x, f64p), ptr(d, f64p)))
        return d, g.reshape(J, J), x

    def partial_reconstruct(self, coords, mode: int, j: int) -> np.ndarray:
        """partial_reconstruct (tucker_model.hpp:136-154) at each coordinate."""
        c = np.ascontiguousarray(coords, np.uint32).reshape(-1)
        if c.size % self.order:
            raise ValueError("coordinate buffer must hold order() values per query")
        nq = c.size // self.order
        out = np.zeros(max(nq, 1))
        check(self._L.vest_partial_reconstruct(self.h, ptr(c, u32p), nq, mode, j, ptr(out, f64p)))
        return out[:nq]

    def get_factor_rows(self, mode: int, lo: int, n: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = np.zeros((n, self.ranks[mode])) if out is None else out
        check(self._L.vest_get_factor_rows(self.h, mode, lo, n, ptr(out, f64p)))
        return out

    def predict(self, coords) -> np.ndarray:
        c = np.ascontiguousarray(coords, np.uint32).reshape(-1)
        if c.size % self.order:
            raise ValueError("coordinate buffer must hold order() values per query")
        nq = c.size // self.order
        out = np.zeros(max(nq, 1))
        check(self._L.vest_predict(self.h, ptr(c, u32p), nq, ptr(out, f64p)))
        return out[:nq]

    def evaluate(self, test: SparseTensor) -> float:
        c = np.ascontiguousarray(test.coords, np.uint32).reshape(-1)
        v = np.ascontiguousarray(test.values, np.float64)
        re = C.c_double()
        check(self._L.vest_evaluate(self.h, ptr(c, u32p), ptr(v, f64p), test.nnz(), C.byref(re)))
        return re.value

    def compute_responsibilities(self, want: bool = True) -> ResponsibilityTable:
        base = C.c_double()
        if not want:
            check(self._L.vest_compute_responsibilities(self.h, None, None, C.byref(base)))
            return ResponsibilityTable(None, None, base.value)
        core = np.zeros(int(np.prod(self.ranks)))
        fs = [np.zeros(d * r) for d, r in zip(self.dims, self.ranks)]
        fp = (f64p * self.order)(*[ptr(f, f64p) for f in fs])
        check(self._L.vest_compute_responsibilities(self.h, ptr(core, f64p), fp, C.byref(base)))
        return ResponsibilityTable(core, fs, base.value)

    def prune_step(self, pr: float, table: Optional[ResponsibilityTable] = None) -> PruneCounts:
        counts = np.zeros(1 + self.order, np.uint64)
        if table is None or table.core is None:
            check(self._L.vest_prune_step(self.h, float(pr), None, None, ptr(counts, u64p)))
        else:
            core = np.ascontiguousarray(table.core, np.float64)
            fs = [np.ascontiguousarray(f, np.float64).reshape(-1) for f in table.factors]
            fp = (f64p * self.order)(*[ptr(f, f64p) for f in fs])
            check(self._L.vest_prune_step(self.h, float(pr), ptr(core, f64p), fp, ptr(counts, u64p)))
        return PruneCounts(int(counts[0]), [int(c) for c in counts[1:]])

    def sparsity(self):
        z, m = C.c_double(), C.c_double()
        check(self._L.vest_sparsity(self.h, C.byref(z), C.byref(m)))
        return z.value, m.value

    def normalize_columns(self):
        check(self._L.vest_normalize_columns(self.h))


def _fingerprint(x: SparseTensor) -> bytes:
    h = hashlib.blake2b(digest_size=16)
    h.update(np.ascontiguousarray(x.coords).view(np.uint8).reshape(-1))
    h.update(np.ascontiguousarray(x.values).view(np.uint8).reshape(-1))
    return h.digest()


def _tensor_device(x: SparseTensor, ranks) -> Device:
    """The tensor's cached device context; rebuilt when the tensor's contents
    changed since it was built (in-place edits of coords/values)."""
    key = tuple(int(r) for r in ranks)
    fp = _fingerprint(x)
    hit = x._devices.get(key)
    if hit is not None and hit[1] != fp:
        hit[0].close()
        hit = None
    if hit is None:
        hit = (Device(x, key), fp)
        x._devices[key] = hit
    return hit[0]


_model_devices: dict = {}


def _model_device(m: TuckerModel) -> Device:
    """A context without observed entries, for model-only operations."""
    key = (tuple(m.dims), tuple(m.ranks))
    dev = _model_devices.get(key)
    if dev is None:
        empty = SparseTensor(list(m.dims), np.zeros((0, m.order()), np.uint32), np.zeros(0))
        dev = Device(empty, m.ranks)
        _model_devices[key] = dev
    return dev


def _bind(m: TuckerModel, x: SparseTensor) -> Device:
    if list(m.dims) != list(x.dims):
        raise ValueError("model/tensor shape mismatch")
    dev = _tensor_device(x, m.ranks)
    dev.set_model(m)
    return dev


# ------------------------------------------------- reference-signature mirror --
def compute_delta(m: TuckerModel, at, mode: int) -> np.ndarray:
    """compute_delta (updates.hpp:35-59)."""
    dev = _model_device(m)
    dev.set_model(m)
    return dev.compute_delta(at, mode)


def reconstruct_entry(m: TuckerModel, at) -> float:
    """reconstruct_entry (tucker_model.hpp:112-131)."""
    return float(predict(m, np.asarray(at, np.uint32).reshape(1, -1))[0])


def partial_reconstruct(m: TuckerModel, at, mode: int, j: int) -> float:
    """partial_reconstruct (tucker_model.hpp:136-154)."""
    dev = _model_device(m)
    dev.set_model(m)
    return float(dev.partial_reconstruct(np.asarray(at, np.uint32).reshape(1, -1), mode, j)[0])


class RowUpdateScratch:
    """RowUpdateScratch (updates.hpp:17-30)."""

    def __init__(self):
        self.delta = np.zeros(0)
        self.gram = np.zeros(0)
        self.xdelta = np.zeros(0)

    def reset(self, J: int):
        self.delta = np.zeros(J)
        self.gram = np.zeros(J * J)
        self.xdelta = np.zeros(J)


def _row_stats_into(dev: Device, mode: int, i: int, s: RowUpdateScratch):
    d, g, x = dev.row_stats(mode, i)
    s.delta, s.gram, s.xdelta = d, g.reshape(-1), x


def compute_row_stats(m, x, idx, mode: int, i: int, s: RowUpdateScratch):
    """compute_row_stats (updates.hpp:64-79), bit-identical."""
    if not (0 <= mode < m.order() and 0 <= i < m.dims[mode]):
        raise ValueError("row out of range")
    _row_stats_into(_bind(m, x), mode, i, s)


def _row_update(m, x, idx, mode, i, lam, reg, s):
    if not (0 <= mode < m.order() and 0 <= i < m.dims[mode]):
        raise ValueError("row out of range")
    if reg == Regularizer.LF and s is not None and idx is not None and len(idx.slice(mode, i)) == 0:
        return  # updates.hpp:91: the scratch is not touched either
    dev = _bind(m, x)
    if s is not None:
        _row_stats_into(dev, mode, i, s)
    dev.update_factor_row(reg, mode, i, lam)
    f = m.factors[mode]
    dev.get_factor_rows(mode, i, 1, out=f[i:i + 1])  # only this row changed


def update_factor_row_lf(m, x, idx, mode, i, lam, s: Optional[RowUpdateScratch] = None):
    """update_factor_row_lf (updates.hpp:88-106, :141-145); with `s` the
    scratch overload (the row's statistics are left in s)."""
    _row_update(m, x, idx, mode, i, lam, Regularizer.LF, s)


def update_factor_row_l1(m, x, idx, mode, i, lam, s: Optional[RowUpdateScratch] = None):
    """update_factor_row_l1 (updates.hpp:113-139, :147-151)."""
    _row_update(m, x, idx, mode, i, lam, Regularizer.L1, s)


def update_all_factors(m, x, idx, reg, lam, threads: int = 1):
    """update_all_factors (updates.hpp:157-175); `threads` is accepted and ignored."""
    dev = _bind(m, x)
    dev.update_all_factors(reg, lam)
    dev.get_model(into=m)


def update_core_lf(m, x, lam, threads: int = 1):
    """update_core_lf (updates.hpp:253-256)."""
    dev = _bind(m, x)
    dev.update_core(Regularizer.LF, lam)
    dev.get_model(into=m)


def update_core_l1(m, x, lam, threads: int = 1):
    """update_core_l1 (updates.hpp:259-262)."""
    dev = _bind(m, x)
    dev.update_core(Regularizer.L1, lam)
    dev.get_model(into=m)


def compute_residuals(m, x, threads: int = 1) -> Residuals:
    """compute_residuals (tucker_model.hpp:168-183)."""
    dev = _bind(m, x)
    return dev.compute_residuals(want_r=True)


def reconstruction_error(m, x) -> float:
    """reconstruction_error (tucker_model.hpp:186-188)."""
    dev = _bind(m, x)
    return dev.compute_residuals().re


def compute_responsibilities(m, x, idx, res: Residuals, threads: int = 1) -> ResponsibilityTable:
    """compute_responsibilities (pruning.hpp:181-191).  The residual used is the
    device residual of `m` on `x` -- the only residual the reference ever passes
    here (trainer.hpp:127,136)."""
    dev = _bind(m, x)
    return dev.compute_responsibilities()


def compute_core_responsibilities(m, x, res: Residuals, threads: int = 1) -> np.ndarray:
    """compute_core_responsibilities (pruning.hpp:98-134)."""
    return compute_responsibilities(m, x, None, res, threads).core


def compute_factor_responsibilities(m, x, idx, mode: int, res: Residuals, threads: int = 1) -> np.ndarray:
    """compute_factor_responsibilities (pruning.hpp:141-179)."""
    return compute_responsibilities(m, x, idx, res, threads).factors[mode]


def prune_step(m: TuckerModel, table: ResponsibilityTable, pr: float) -> PruneCounts:
    """prune_step (pruning.hpp:234-247): device radix select per block."""
    if not (pr >= 0.0 and pr < 1.0):
        raise ValueError("prune rate must be in [0, 1)")
    dev = _model_device(m)
    dev.set_model(m)
    counts = dev.prune_step(pr, table)
    dev.get_model(into=m)
    return counts


def sparsity(m: TuckerModel) -> float:
    """sparsity (tucker_model.hpp:192-198)."""
    dev = _model_device(m)
    dev.set_model(m)
    return dev.sparsity()[0]


def masked_fraction(m: TuckerModel) -> float:
    """masked_fraction (tucker_model.hpp:201-207)."""
    dev = _model_device(m)
    dev.set_model(m)
    return dev.sparsity()[1]


def normalize_columns(m: TuckerModel) -> None:
    """normalize_columns (tucker_model.hpp:212-236)."""
    dev = _model_device(m)
    dev.set_model(m)
    dev.normalize_columns()
    dev.get_model(into=m)


def predict(m: TuckerModel, flat_coords) -> np.ndarray:
    """predict (trainer.hpp:172-185)."""
    c = np.ascontiguousarray(flat_coords, np.uint32).reshape(-1)
    if m.order() == 0 or c.size % m.order():
        raise ValueError("coordinate buffer must hold order() values per query")
    dev = _model_device(m)
    dev.set_model(m)
    return dev.predict(c)


def evaluate_test(m: TuckerModel, test: SparseTensor) -> float:
    """evaluate_test (trainer.hpp:188-190)."""
    if list(m.dims) != list(test.dims):
        raise ValueError("model/tensor shape mismatch")
    dev = _model_device(m)
    dev.set_model(m)
    return dev.evaluate(test)


def save_model(m: "TuckerModel", dir_path) -> None:
    """save_model (model_io.hpp:22-51): factor_<n>.tsv + core.coo, byte-identical."""
    d = np.asarray(m.dims, np.uint64)
    r = np.asarray(m.ranks, np.uint64)
    core = np.ascontiguousarray(m.core, np.float64).reshape(-1)
    fs = [np.ascontiguousarray(f, np.float64).reshape(-1) for f in m.factors]
    fp = (f64p * len(fs))(*[ptr(f, f64p) for f in fs])
    _lib.io_check(_lib.lib().vest_model_save(str(dir_path).encode(), len(fs), ptr(d, u64p), ptr(r, u64p),
                                             ptr(core, f64p), fp))


def load_model(dir_path) -> "TuckerModel":
    """load_model (model_io.hpp:53-104): every zero element is pruned."""
    L = _lib.lib()
    h = C.c_void_p()
    _lib.io_check(L.vest_model_load(str(dir_path).encode(), C.byref(h)))
    try:
        order = C.c_int()
        _lib.io_check(L.vest_model_file_info(h, C.byref(order), None, None, None, None, None, None))
        n = order.value
        dims = np.zeros(n, np.uint64)
        ranks = np.zeros(n, np.uint64)
        cp, cmp_ = f64p(), u8p()
        fps = (f64p * n)()
        mps = (u8p * n)()
        _lib.io_check(L.vest_model_file_info(h, None, ptr(dims, u64p), ptr(ranks, u64p), C.byref(cp), C.byref(cmp_),
                                             fps, mps))
        dims_l, ranks_l = [int(v) for v in dims], [int(v) for v in ranks]
        G = int(np.prod(ranks_l))
        core = np.ctypeslib.as_array(cp, shape=(G,)).copy()
        core_mask = np.ctypeslib.as_array(cmp_, shape=(G,)).copy()
        factors = [np.ctypeslib.as_array(fps[k], shape=(dims_l[k] * ranks_l[k],)).copy().reshape(dims_l[k], ranks_l[k])
                   for k in range(n)]
        masks = [np.ctypeslib.as_array(mps[k], shape=(dims_l[k] * ranks_l[k],)).copy().reshape(dims_l[k], ranks_l[k])
                 for k in range(n)]
        return TuckerModel(dims_l, ranks_l, core, core_mask, factors, masks)
    finally:
        L.vest_model_file_free(h)


def split_train_test(x: SparseTensor, test_fraction: float, seed: int):
    """split_train_test (sparse_tensor.hpp:232-260)."""
    if not (test_fraction >= 0.0 and test_fraction <= 1.0):
        raise ValueError("test_fraction must be in [0, 1]")
    n = x.nnz()
    te = np.zeros(max(n, 1), np.uint64)
    tr = np.zeros(max(n, 1), np.uint64)
    nte, ntr = C.c_uint64(), C.c_uint64()
    check(_lib.lib().vest_split_ids(n, float(test_fraction), seed, ptr(te, u64p), C.byref(nte),
                                    ptr(tr, u64p), C.byref(ntr)))
    te, tr = te[: nte.value], tr[: ntr.value]
    mk = lambda ids: SparseTensor(list(x.dims), x.coords[ids.astype(np.int64)], x.values[ids.astype(np.int64)])
    return mk(tr), mk(te)


# -------------------------------------------------------------- host control --
@dataclass
class PruneSchedule:
    """rate(t) = min(init_pr * t, max_pr) (pruning.hpp:20-33)."""

    init_pr: float = 0.01
    max_pr: float = 0.1

    def validate(self):
        if not (self.init_pr > 0.0 and self.init_pr <= self.max_pr and self.max_pr < 1.0):
            raise ValueError("require 0 < init_pr <= max_pr < 1")

    def rate(self, it: int) -> float:
        if it == 0:
            raise ValueError("iterations are 1-based")
        return min(self.init_pr * float(it), self.max_pr)


class StopController:
    """Manual target-sparsity / auto elbow stop, latching (pruning.hpp:45-81)."""

    def __init__(self, mode: StopMode = StopMode.Manual, target_sparsity: float = 0.0,
                 elbow_threshold: float = 0.05):
        self.mode = mode
        self.target_sparsity = target_sparsity
        self.elbow_threshold = elbow_threshold
        self._stopped = False
        self._history: list = []

    def should_prune(self, current_sparsity: float, re: float, pr: float) -> bool:
        if self._stopped:
            return False
        if re == 0.0:
            return False
        if self.mode == StopMode.Manual:
            if current_sparsity >= self.target_sparsity:
                self._stopped = True
                return False
            return True
        if len(self._history) >= 2:
            prev = self._history[-1]
            prev2 = self._history[-2]
            stat = (re + prev2 - 2.0 * prev) / pr
            if stat > self.elbow_threshold:
                self._stopped = True
                return False
        return True

    def record_prune_event(self, re: float):
        self._history.append(re)

    def stopped(self) -> bool:
        return self._stopped


@dataclass
class TrainConfig:  # trainer.hpp:31-46
    ranks: list = field(default_factory=list)
    reg: Regularizer = Regularizer.LF
    lam: float = 0.01
    mode: StopMode = StopMode.Manual
    target_sparsity: float = 0.0
    elbow_threshold: float = 0.05
    schedule: PruneSchedule = field(default_factory=PruneSchedule)
    max_iters: int = 100
    tol: float = 1e-4
    threads: int = 0
    seed: int = 0
    normalize_output: bool = True


@dataclass
class IterationReport:  # trainer.hpp:51-61
    iter: int = 0
    re: float = 0.0
    prune_rate: float = 0.0
    pruned: bool = False
    pruned_core: int = 0
    pruned_factors: list = field(default_factory=list)
    sparsity: float = 0.0
    masked: float = 0.0
    wall_ms: float = 0.0


@dataclass
class TrainReport:  # trainer.hpp:63-71
    iterations: list = field(default_factory=list)
    converged: bool = False
    iters: int = 0
    final_re: float = 0.0
    final_sparsity: float = 0.0
    final_masked: float = 0.0
    elapsed_sec: float = 0.0


@dataclass
class FitResult:
    model: TuckerModel
    report: TrainReport


def _check_config(x: SparseTensor, cfg: TrainConfig):
    """detail::check_config (trainer.hpp:80-93)."""
    if len(cfg.ranks) != x.order():
        raise ValueError("ranks order mismatch")
    if any(int(r) == 0 for r in cfg.ranks):
        raise ValueError("ranks must be positive")
    if not (cfg.lam >= 0.0):
        raise ValueError("lambda must be nonnegative")
    if not (cfg.tol >= 0.0):
        raise ValueError("tol must be nonnegative")
    if cfg.max_iters == 0:
        raise ValueError("max_iters must be positive")
    if not (cfg.target_sparsity >= 0.0 and cfg.target_sparsity < 1.0):
        raise ValueError("target sparsity must be in [0, 1)")
    cfg.schedule.validate()
    if x.nnz() == 0:
        raise ValueError("empty tensor")
    if x.frobenius_norm() == 0.0:
        raise ValueError("tensor values are all zero; nothing to fit")


def fit(x: SparseTensor, cfg: TrainConfig, device: int = 0) -> FitResult:
    """fit (trainer.hpp:103-168), device-resident: the model stays in HBM for the
    whole loop; per iteration the host reads back only re, sparsity and prune
    counts for the stop controller."""
    _check_config(x, cfg)
    t_start = time.perf_counter()
    dev = Device(x, cfg.ranks, device)
    dev.init_random(cfg.seed)
    ctrl = StopController(cfg.mode, cfg.target_sparsity, cfg.elbow_threshold)
    report = TrainReport()
    prev_re = math.inf
    for t in range(1, cfg.max_iters + 1):
        it_start = time.perf_counter()
        re = dev.cd_iteration(cfg.reg, cfg.lam)
        pr = cfg.schedule.rate(t)
        rec = IterationReport(iter=t, re=re, prune_rate=pr, pruned_factors=[0] * x.order())
        if ctrl.should_prune(dev.sparsity()[0], re, pr):
            dev.compute_responsibilities(want=False)
            counts = dev.prune_step(pr)
            if counts.total() > 0:
                ctrl.record_prune_event(re)
                rec.pruned = True
                rec.pruned_core = counts.core
                rec.pruned_factors = counts.factors
        rec.sparsity, rec.masked = dev.sparsity()
        rec.wall_ms = (time.perf_counter() - it_start) * 1e3
        report.iterations.append(rec)
        if abs(prev_re - re) < cfg.tol:
            report.converged = True
            break
        prev_re = re
    if cfg.normalize_output:
        dev.normalize_columns()
    report.iters = len(report.iterations)
    report.final_re = dev.compute_residuals().re
    report.final_sparsity, report.final_masked = dev.sparsity()
    model = dev.get_model()
    report.elapsed_sec = time.perf_counter() - t_start
    dev.close()
    return FitResult(model, report)


@dataclass
class RateResult:
    rate: float
    pruned: PruneCounts
    sparsity: float
    train_re: float
    test_re: float


def auto_search(x_train: SparseTensor, x_test: SparseTensor, model: TuckerModel, rates: Sequence[float],
                device: int = 0, dev: Optional["Device"] = None) -> list:
    """Prune-rate sweep (BASELINE config 5; SURVEY App. C option (i)): for each
    rate, start from the trained model, score responsibilities on the training
    entries (pruning.hpp:181-191), prune_step(rate) (pruning.hpp:234-247) and
    evaluate the relative error on the training and held-out entries
    (tucker_model.hpp:186-188, trainer.hpp:188-190).  Device-resident: every
    rate starts from the same model, so its responsibility table is scored
    once and reused; the model is re-uploaded per rate; the evaluation is the
    inner loop.  `dev` reuses a context already built on x_train."""
    own = dev is None
    if own:
        dev = Device(x_train, model.ranks, device)
    dev.set_model(model)
    table = dev.compute_responsibilities()
    out = []
    for pr in rates:
        dev.set_model(model)
        counts = dev.prune_step(float(pr), table)
        train_re = dev.compute_residuals().re
        test_re = dev.evaluate(x_test)
        out.append(RateResult(float(pr), counts, dev.sparsity()[0], train_re, test_re))
    if own:
        dev.close()
    return out
