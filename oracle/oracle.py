"""TEST INFRASTRUCTURE: ctypes bindings for the two CPU oracles.

* kind="port"      -> oracle/libvest_oracle.so (our C restatement, vest_oracle.c)
* kind="reference" -> oracle/_ref/libsparsetuck_ref.so (the unmodified reference
                      headers behind ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs import this module.  The product package never does.

Both libraries export the same session API (vo_* / vr_*), so `Session` drives
either one with identical calls.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libvest_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsetuck_ref.so")

_libs: dict[str, C.CDLL] = {}

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


def build() -> None:
    """Compile the oracles (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


def _lib(kind: str) -> tuple[C.CDLL, str]:
    if kind not in _libs:
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        lib = C.CDLL(path)
        p = "vo_" if kind == "port" else "vr_"
        vp = C.c_void_p
        sig = {
            "last_error": (C.c_char_p, []),
            "create": (C.c_int, [C.c_int, _u64p, C.c_uint64, _u32p, _f64p, _u64p, C.POINTER(vp)]),
            "destroy": (None, [vp]),
            "init_random": (C.c_int, [vp, C.c_uint64]),
            "set_model": (C.c_int, [vp, _f64p, _u8p, C.POINTER(_f64p), C.POINTER(_u8p)]),
            "get_model": (C.c_int, [vp, _f64p, _u8p, C.POINTER(_f64p), C.POINTER(_u8p)]),
            "get_index": (C.c_int, [vp, C.c_int, _u64p, _u32p]),
            "compute_delta": (C.c_int, [vp, _u32p, C.c_int, _f64p]),
            "reconstruct": (C.c_int, [vp, _u32p, C.c_uint64, _f64p]),
            "update_factor_row": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint64, C.c_double]),
            "update_all_factors": (C.c_int, [vp, C.c_int, C.c_double, C.c_int]),
            "update_core": (C.c_int, [vp, C.c_int, C.c_double, C.c_int]),
            "compute_residuals": (C.c_int, [vp, C.c_int, _f64p, _f64p, _f64p, _f64p]),
            "compute_responsibilities": (C.c_int, [vp, C.c_int, _f64p, C.POINTER(_f64p)]),
            "prune_step": (C.c_int, [vp, C.c_double, _f64p, C.POINTER(_f64p), _u64p]),
            "sparsity": (C.c_double, [vp]),
            "masked_fraction": (C.c_double, [vp]),
            "normalize_columns": (C.c_int, [vp]),
            "frobenius_norm": (C.c_double, [vp]),
            "cd_iteration": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, _f64p]),
            "row_stats": (C.c_int, [vp, C.c_int, C.c_uint64, _f64p, _f64p, _f64p]),
            "partial_reconstruct": (C.c_int, [vp, _u32p, C.c_uint64, C.c_int, C.c_uint64, _f64p]),
        }
        if kind == "port":
            sig["update_factor_mode"] = (C.c_int, [vp, C.c_int, C.c_int, C.c_double, C.c_int])
        for name, (res, args) in sig.items():
            fn = getattr(lib, p + name)
            fn.restype = res
            fn.argtypes = args
        if kind == "reference":
            lib.vr_split_ids.restype = C.c_int
            lib.vr_split_ids.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _u64p, _u64p, _u64p, _u64p]
            lib.vr_fit.restype = C.c_int
            lib.vr_fit.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_uint64,
                                   C.c_int, C.c_int, _f64p, _u8p, _f64p, _u64p, _f64p]
        _libs[kind] = (lib, p)
    return _libs[kind]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class OracleError(Exception):
    pass


class Session:
    """One tensor + model, driven through the oracle's session API."""

    def __init__(self, dims, coords, values, ranks, kind: str = "port"):
        self.kind = kind
        self.lib, self.p = _lib(kind)
        self.dims = np.ascontiguousarray(dims, dtype=np.uint64)
        self.ranks = np.ascontiguousarray(ranks, dtype=np.uint64)
        self.order = len(self.dims)
        self.coords = np.ascontiguousarray(coords, dtype=np.uint32).reshape(-1)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.nnz = len(self.values)
        h = C.c_void_p()
        rc = self._f("create")(self.order, _ptr(self.dims, _u64p), self.nnz,
                               _ptr(self.coords, _u32p), _ptr(self.values, _f64p),
                               _ptr(self.ranks, _u64p), C.byref(h))
        self._check(rc)
        self.h = h

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc != 0:
            msg = self._f("last_error")().decode()
            raise (ValueError if rc == 1 else OracleError)(msg)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self._f("destroy")(h)
            self.h = None

    # ---- model -------------------------------------------------------------
    def core_size(self) -> int:
        return int(np.prod(self.ranks))

    def init_random(self, seed: int):
        self._check(self._f("init_random")(self.h, seed))

    def set_model(self, core, core_mask, factors, factor_masks):
        core = np.ascontiguousarray(core, np.float64)
        cm = np.ascontiguousarray(core_mask, np.uint8)
        fs = [np.ascontiguousarray(f, np.float64).reshape(-1) for f in factors]
        ms = [np.ascontiguousarray(m, np.uint8).reshape(-1) for m in factor_masks]
        fp = (_f64p * self.order)(*[_ptr(f, _f64p) for f in fs])
        mp = (_u8p * self.order)(*[_ptr(m, _u8p) for m in ms])
        self._check(self._f("set_model")(self.h, _ptr(core, _f64p), _ptr(cm, _u8p), fp, mp))

    def get_model(self):
        core = np.zeros(self.core_size(), np.float64)
        cm = np.zeros(self.core_size(), np.uint8)
        fs = [np.zeros((int(d), int(r)), np.float64) for d, r in zip(self.dims, self.ranks)]
        ms = [np.zeros((int(d), int(r)), np.uint8) for d, r in zip(self.dims, self.ranks)]
        fp = (_f64p * self.order)(*[_ptr(f, _f64p) for f in fs])
        mp = (_u8p * self.order)(*[_ptr(m, _u8p) for m in ms])
        self._check(self._f("get_model")(self.h, _ptr(core, _f64p), _ptr(cm, _u8p), fp, mp))
        return core, cm, fs, ms

    def get_index(self, mode: int):
        off = np.zeros(int(self.dims[mode]) + 1, np.uint64)
        ids = np.zeros(max(self.nnz, 1), np.uint32)
        self._check(self._f("get_index")(self.h, mode, _ptr(off, _u64p), _ptr(ids, _u32p)))
        return off, ids[: self.nnz]

    # ---- kernels -----------------------------------------------------------
    def compute_delta(self, at, mode: int):
        at = np.ascontiguousarray(at, np.uint32)
        out = np.zeros(int(self.ranks[mode]), np.float64)
        self._check(self._f("compute_delta")(self.h, _ptr(at, _u32p), mode, _ptr(out, _f64p)))
        return out

    def reconstruct(self, coords):
        c = np.ascontiguousarray(coords, np.uint32).reshape(-1)
        nq = len(c) // self.order
        out = np.zeros(max(nq, 1), np.float64)
        self._check(self._f("reconstruct")(self.h, _ptr(c, _u32p), nq, _ptr(out, _f64p)))
        return out[:nq]

    def update_factor_row(self, reg: int, mode: int, row: int, lam: float):
        self._check(self._f("update_factor_row")(self.h, reg, mode, row, lam))

    def update_factor_mode(self, reg: int, mode: int, lam: float, threads: int = 1):
        """One mode of update_all_factors (port only)."""
        self._check(self._f("update_factor_mode")(self.h, reg, mode, lam, threads))

    def row_stats(self, mode: int, row: int):
        """compute_row_stats (updates.hpp:64-79) -> (delta, gram J x J, xdelta)."""
        J = int(self.ranks[mode])
        d, g, x = np.zeros(J), np.zeros(J * J), np.zeros(J)
        self._check(self._f("row_stats")(self.h, mode, row, _ptr(d, _f64p), _ptr(g, _f64p), _ptr(x, _f64p)))
        return d, g.reshape(J, J), x

    def partial_reconstruct(self, coords, mode: int, j: int):
        c = np.ascontiguousarray(coords, np.uint32).reshape(-1)
        nq = len(c) // self.order
        out = np.zeros(max(nq, 1), np.float64)
        self._check(self._f("partial_reconstruct")(self.h, _ptr(c, _u32p), nq, mode, j, _ptr(out, _f64p)))
        return out[:nq]

    def update_all_factors(self, reg: int, lam: float, threads: int = 1):
        self._check(self._f("update_all_factors")(self.h, reg, lam, threads))

    def update_core(self, reg: int, lam: float, threads: int = 1):
        self._check(self._f("update_core")(self.h, reg, lam, threads))

    def compute_residuals(self, threads: int = 1, want_r: bool = True):
        r = np.zeros(max(self.nnz, 1), np.float64) if want_r else None
        ss, xn, re = C.c_double(), C.c_double(), C.c_double()
        self._check(self._f("compute_residuals")(
            self.h, threads, _ptr(r, _f64p) if want_r else None, C.byref(ss), C.byref(xn), C.byref(re)))
        return (r[: self.nnz] if want_r else None), ss.value, xn.value, re.value

    def compute_responsibilities(self, threads: int = 1):
        core = np.zeros(self.core_size(), np.float64)
        fs = [np.zeros(int(d) * int(r), np.float64) for d, r in zip(self.dims, self.ranks)]
        fp = (_f64p * self.order)(*[_ptr(f, _f64p) for f in fs])
        self._check(self._f("compute_responsibilities")(self.h, threads, _ptr(core, _f64p), fp))
        return core, fs

    def prune_step(self, pr: float, core_resp=None, factor_resp=None):
        counts = np.zeros(1 + self.order, np.uint64)
        if core_resp is None:
            self._check(self._f("prune_step")(self.h, pr, None, None, _ptr(counts, _u64p)))
        else:
            cr = np.ascontiguousarray(core_resp, np.float64)
            frs = [np.ascontiguousarray(f, np.float64).reshape(-1) for f in factor_resp]
            fp = (_f64p * self.order)(*[_ptr(f, _f64p) for f in frs])
            self._check(self._f("prune_step")(self.h, pr, _ptr(cr, _f64p), fp, _ptr(counts, _u64p)))
        return counts

    def sparsity(self) -> float:
        return self._f("sparsity")(self.h)

    def masked_fraction(self) -> float:
        return self._f("masked_fraction")(self.h)

    def normalize_columns(self):
        self._check(self._f("normalize_columns")(self.h))

    def frobenius_norm(self) -> float:
        return self._f("frobenius_norm")(self.h)

    def cd_iteration(self, reg: int, lam: float, threads: int = 1) -> float:
        re = C.c_double()
        self._check(self._f("cd_iteration")(self.h, reg, lam, threads, C.byref(re)))
        return re.value


def split_ids(nnz: int, test_fraction: float, seed: int):
    """Reference split_train_test entry ids (reference library only)."""
    lib, _ = _lib("reference")
    te = np.zeros(max(nnz, 1), np.uint64)
    tr = np.zeros(max(nnz, 1), np.uint64)
    nte, ntr = C.c_uint64(), C.c_uint64()
    rc = lib.vr_split_ids(nnz, test_fraction, seed, _ptr(te, _u64p), C.byref(nte), _ptr(tr, _u64p), C.byref(ntr))
    if rc:
        raise ValueError(lib.vr_last_error().decode())
    return te[: nte.value], tr[: ntr.value]
