"""ctypes loader for libvest_cuda.so (the C-ABI in include/vest.h).

The product path has no CPU fallback: if the shared library is missing the
import of any compute entry point raises.  The library itself loads on a
machine without a GPU (CUDA is only touched when a context is created), which
lets the CPU test-suite check its exported symbols.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VEST_LIB") or os.path.join(HERE, "libvest_cuda.so")
CSRC = os.path.join(HERE, "csrc")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p

# name -> (restype, argtypes); mirrors include/vest.h
SIGNATURES = {
    "vest_last_error": (C.c_char_p, []),
    "vest_version": (C.c_char_p, []),
    "vest_launch_count": (C.c_uint64, []),
    "vest_ctx_create": (C.c_int, [C.c_int, u64p, C.c_uint64, u32p, f64p, u64p, C.c_int, C.POINTER(vp)]),
    "vest_ctx_destroy": (C.c_int, [vp]),
    "vest_ctx_stream": (vp, [vp]),
    "vest_ctx_device_bytes": (C.c_uint64, [vp]),
    "vest_ctx_specialised": (C.c_int, [vp]),
    "vest_ctx_force_generic": (C.c_int, [vp, C.c_int]),
    "vest_ctx_set_core_block": (C.c_int, [vp, C.c_int]),
    "vest_ctx_set_sparse_delta": (C.c_int, [vp, C.c_int]),
    "vest_ctx_sparse_delta_active": (C.c_int, [vp]),
    "vest_ctx_set_core_gen": (C.c_int, [vp, C.c_int]),
    "vest_sparse_compile_check": (C.c_int, [C.c_int, u64p, u8p, u64p]),
    "vest_init_random": (C.c_int, [vp, C.c_uint64]),
    "vest_init_random_host": (C.c_int, [C.c_int, u64p, u64p, C.c_uint64, f64p, C.POINTER(f64p)]),
    "vest_get_mode_index": (C.c_int, [vp, C.c_int, u64p, u32p]),
    "vest_set_model": (C.c_int, [vp, f64p, u8p, C.POINTER(f64p), C.POINTER(u8p)]),
    "vest_get_model": (C.c_int, [vp, f64p, u8p, C.POINTER(f64p), C.POINTER(u8p)]),
    "vest_update_all_factors": (C.c_int, [vp, C.c_int, C.c_double]),
    "vest_update_factor_mode": (C.c_int, [vp, C.c_int, C.c_int, C.c_double]),
    "vest_update_factor_row": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint64, C.c_double]),
    "vest_update_core": (C.c_int, [vp, C.c_int, C.c_double]),
    "vest_compute_residuals": (C.c_int, [vp, f64p, f64p, f64p, f64p]),
    "vest_cd_iteration": (C.c_int, [vp, C.c_int, C.c_double, f64p]),
    "vest_cd_iteration_host": (C.c_int, [vp, f64p, u8p, C.POINTER(f64p), C.POINTER(u8p), C.c_int, C.c_double,
                                         f64p]),
    "vest_compute_delta": (C.c_int, [vp, u32p, C.c_int, f64p]),
    "vest_predict": (C.c_int, [vp, u32p, C.c_uint64, f64p]),
    "vest_ctx_set_gather_f32": (C.c_int, [vp, C.c_int]),
    "vest_ctx_set_sparse_fused": (C.c_int, [vp, C.c_int]),
    "vest_compute_row_stats": (C.c_int, [vp, C.c_int, C.c_uint64, f64p, f64p, f64p]),
    "vest_partial_reconstruct": (C.c_int, [vp, u32p, C.c_uint64, C.c_int, C.c_uint64, f64p]),
    "vest_get_factor_rows": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, f64p]),
    "vest_evaluate": (C.c_int, [vp, u32p, f64p, C.c_uint64, f64p]),
    "vest_compute_responsibilities": (C.c_int, [vp, f64p, C.POINTER(f64p), f64p]),
    "vest_prune_step": (C.c_int, [vp, C.c_double, f64p, C.POINTER(f64p), u64p]),
    "vest_sparsity": (C.c_int, [vp, f64p, f64p]),
    "vest_normalize_columns": (C.c_int, [vp]),
    "vest_frobenius_norm": (C.c_int, [vp, f64p]),
    "vest_ctx_profile": (C.c_int, [vp, C.c_int]),
    "vest_ctx_profile_read": (C.c_int, [vp, f64p, u64p, C.c_int]),
    "vest_measure_fp64_peak": (C.c_int, [C.c_int, f64p]),
    "vest_ctx_create_shard": (C.c_int, [C.c_int, u64p, C.c_uint64, u32p, f64p, u64p, C.c_int, u64p, u64p,
                                        C.POINTER(vp)]),
    "vest_ctx_set_comm": (C.c_int, [vp, vp]),
    "vest_ctx_local_nnz": (C.c_uint64, [vp, C.c_int]),
    "vest_synth": (C.c_int, [C.c_int, u64p, C.c_uint64, f64p, C.c_int, C.c_uint64, u32p, f64p]),
    "vest_split_ids": (C.c_int, [C.c_uint64, C.c_double, C.c_uint64, u64p, u64p, u64p, u64p]),
    "vest_partition_rows": (C.c_int, [u64p, C.c_uint64, C.c_int, u64p]),
    "vest_nccl_unique_id": (C.c_int, [vp]),
    "vest_ctx_set_nccl": (C.c_int, [vp, C.c_int, C.c_int, vp, u64p]),
    # data formats (vest_io.cpp)
    "vest_io_last_error": (C.c_char_p, []),
    "vest_coo_load": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]),
    "vest_coo_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_uint64), u64p, C.POINTER(u32p),
                                C.POINTER(f64p)]),
    "vest_coo_free": (None, [vp]),
    "vest_coo_save": (C.c_int, [C.c_char_p, C.c_int, u64p, C.c_uint64, u32p, f64p]),
    "vest_coo_cache_save": (C.c_int, [C.c_char_p, C.c_int, u64p, C.c_uint64, u32p, f64p]),
    "vest_coo_cache_load": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "vest_model_save": (C.c_int, [C.c_char_p, C.c_int, u64p, u64p, f64p, C.POINTER(f64p)]),
    "vest_model_load": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "vest_model_file_info": (C.c_int, [vp, C.POINTER(C.c_int), u64p, u64p, C.POINTER(f64p), C.POINTER(u8p),
                                       C.POINTER(f64p), C.POINTER(u8p)]),
    "vest_model_file_free": (None, [vp]),
}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile libvest_cuda.so in-tree for sm_100a (nvcc; no GPU needed)."""
    out = subprocess.run(["make", "-s", "-C", CSRC, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("libvest_cuda.so build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if verbose:
        print(out.stdout)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the VeST CUDA path has no CPU fallback; "
                "build it with paper_1904_02603_b200._lib.build() or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class VestError(RuntimeError):
    pass


class CudaError(VestError):
    pass


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().vest_last_error().decode()
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 3:
        raise CudaError(msg)
    raise VestError(msg)  # std::runtime_error


def io_check(rc: int) -> None:
    """Status of a data-format call (vest_io.cpp): the reference's exception
    type and message (std::invalid_argument -> ValueError, std::runtime_error
    -> VestError)."""
    if rc == 0:
        return
    msg = lib().vest_io_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise VestError(msg)


def ptr(a, t):
    return a.ctypes.data_as(t)
