"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref):

    make -C oracle && python tests/golden/make_golden.py

Every fixture is produced by oracle/_ref/libsparsetuck_ref.so, i.e. the
unmodified reference headers (proj/include/sparsetuck/*.hpp) behind
oracle/ref_shim.cpp.  Inputs (coordinates, values) are drawn here with numpy
and stored in the fixture, so the fixtures do not depend on any RNG except the
reference's own init_random (tucker_model.hpp:88-108), whose output is stored
too.

The fixtures pin (a) the C restatement oracle/vest_oracle.c (tests/test_oracle.py,
CPU) and (b) the CUDA path (tests/test_gpu_parity.py, GPU).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def random_tensor(dims, nnz, rng, lo=-1.0, hi=2.0):
    """Distinct coordinates in row-major order, values U[lo, hi)."""
    total = int(np.prod(dims))
    cells = np.sort(rng.choice(total, size=nnz, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    return coords, rng.uniform(lo, hi, nnz)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def sequence_case(name, dims, ranks, nnz, seed, reg, lam, iters, prune_at, pr, data_seed,
                  mask_frac=0.0):
    """init_random -> iters x (factors, core, residuals[, resp + prune])."""
    rng = np.random.default_rng(data_seed)
    coords, values = random_tensor(dims, nnz, rng)
    s = O.Session(dims, coords, values, ranks, "reference")
    s.init_random(seed)
    out = dict(dims=np.array(dims, np.uint64), ranks=np.array(ranks, np.uint64), coords=coords,
               values=values, seed=np.uint64(seed), reg=np.int32(reg), lam=np.float64(lam),
               iters=np.int32(iters), prune_at=np.array(prune_at, np.int32), pr=np.float64(pr))
    core, cm, fs, ms = s.get_model()
    if mask_frac > 0:
        # pre-mask a seeded subset (values zeroed) so kernels see pruned positions
        mrng = np.random.default_rng(data_seed + 1000)
        cmask = (mrng.random(core.shape) < mask_frac).astype(np.uint8)
        core[cmask == 1] = 0.0
        cm = cmask
        for n in range(len(dims)):
            fm = (mrng.random(fs[n].shape) < mask_frac).astype(np.uint8)
            fs[n][fm == 1] = 0.0
            ms[n] = fm
        s.set_model(core, cm, fs, ms)
    out["init_core"], out["init_core_mask"] = core, cm
    for n in range(len(dims)):
        out[f"init_factor{n}"], out[f"init_fmask{n}"] = fs[n], ms[n]
    for n in range(len(dims)):
        off, ids = s.get_index(n)
        out[f"index_offsets{n}"], out[f"index_ids{n}"] = off, ids
    for t in range(1, iters + 1):
        s.update_all_factors(reg, lam, 1)
        _, _, fs, _ = s.get_model()
        for n in range(len(dims)):
            out[f"t{t}_factors_factor{n}"] = fs[n]
        s.update_core(reg, lam, 1)
        core, _, fs, _ = s.get_model()
        out[f"t{t}_core"] = core
        r, ss, xn, re = s.compute_residuals(1)
        out[f"t{t}_r"], out[f"t{t}_sum_sq"], out[f"t{t}_x_norm"], out[f"t{t}_re"] = r, ss, xn, re
        out[f"t{t}_sparsity"] = s.sparsity()
        if t in prune_at:
            rc, rf = s.compute_responsibilities(1)
            out[f"t{t}_resp_core"] = rc
            for n in range(len(dims)):
                out[f"t{t}_resp_factor{n}"] = rf[n]
            counts = s.prune_step(pr)
            out[f"t{t}_prune_counts"] = counts
            core, cm, fs, ms = s.get_model()
            out[f"t{t}_pruned_core"], out[f"t{t}_pruned_core_mask"] = core, cm
            for n in range(len(dims)):
                out[f"t{t}_pruned_factor{n}"], out[f"t{t}_pruned_fmask{n}"] = fs[n], ms[n]
            out[f"t{t}_masked_fraction"] = s.masked_fraction()
    s.normalize_columns()
    core, _, fs, _ = s.get_model()
    out["normalized_core"] = core
    for n in range(len(dims)):
        out[f"normalized_factor{n}"] = fs[n]
    # delta / reconstruct probes on the final model
    probe = coords[: min(8, nnz)]
    out["probe_coords"] = probe
    out["probe_recon"] = s.reconstruct(probe)
    for n in range(len(dims)):
        out[f"probe_delta{n}"] = np.stack([s.compute_delta(c, n) for c in probe])
    save(name, **out)


def init_case():
    out = {}
    for k, (dims, ranks, seed) in enumerate([((5, 4, 3), (2, 3, 2), 11), ((8, 7, 6), (3, 3, 2), 12),
                                              ((30, 20, 10), (5, 5, 5), 3),
                                              ((6, 5, 4, 3), (2, 2, 2, 2), 0)]):
        coords = np.zeros((1, len(dims)), np.uint32)
        s = O.Session(dims, coords, np.ones(1), ranks, "reference")
        s.init_random(seed)
        core, _, fs, _ = s.get_model()
        out[f"case{k}_dims"] = np.array(dims, np.uint64)
        out[f"case{k}_ranks"] = np.array(ranks, np.uint64)
        out[f"case{k}_seed"] = np.uint64(seed)
        out[f"case{k}_core"] = core
        for n in range(len(dims)):
            out[f"case{k}_factor{n}"] = fs[n]
    out["ncases"] = np.int32(4)
    save("init_random", **out)


def split_case():
    te, tr = O.split_ids(1200, 0.1, 5)
    te2, tr2 = O.split_ids(1000, 0.1, 2024)
    save("split", test_1200=te, train_1200=tr, test_1000=te2, train_1000=tr2)


def fit_case():
    """fit() traces (trainer.hpp:103-168): manual and auto stop modes."""
    rng = np.random.default_rng(77)
    dims, ranks = (12, 10, 8), (3, 3, 2)
    coords, values = random_tensor(dims, 300, rng, 0.0, 1.0)
    out = dict(dims=np.array(dims, np.uint64), ranks=np.array(ranks, np.uint64), coords=coords,
               values=values)
    import ctypes as C
    lib, _ = O._lib("reference")
    for tag, auto, target in (("manual", 0, 0.4), ("auto", 1, 0.0)):
        s = O.Session(dims, coords, values, ranks, "reference")
        it = 25
        re = np.zeros(it)
        pruned = np.zeros(it, np.uint8)
        sp = np.zeros(it)
        iters, fre = C.c_uint64(), C.c_double()
        rc = lib.vr_fit(s.h, 0, 0.01, auto, target, 0.05, 0.02, 0.1, it, 1e-7, 5, 1, 1,
                        re.ctypes.data_as(C.POINTER(C.c_double)),
                        pruned.ctypes.data_as(C.POINTER(C.c_uint8)),
                        sp.ctypes.data_as(C.POINTER(C.c_double)), C.byref(iters), C.byref(fre))
        assert rc == 0
        n = iters.value
        out[f"{tag}_re"], out[f"{tag}_pruned"], out[f"{tag}_sparsity"] = re[:n], pruned[:n], sp[:n]
        out[f"{tag}_final_re"] = fre.value
        core, cm, fs, ms = s.get_model()
        out[f"{tag}_core"] = core
        for k in range(len(dims)):
            out[f"{tag}_factor{k}"] = fs[k]
    save("fit_trace", **out)


def main():
    O.build()
    init_case()
    split_case()
    # small instances mirroring the reference test shapes (tests/test_updates.cpp:22-43)
    sequence_case("seq_543_lf", (5, 4, 3), (2, 3, 2), 25, 21, 0, 0.01, 3, (3,), 0.3, 1)
    sequence_case("seq_543_l1_masked", (5, 4, 3), (2, 3, 2), 25, 22, 1, 0.2, 3, (2, 3), 0.2, 2,
                  mask_frac=0.2)
    sequence_case("seq_876_lf", (8, 7, 6), (3, 3, 2), 120, 23, 0, 0.05, 4, (2, 4), 0.25, 3)
    sequence_case("seq_2020_10_lf", (20, 20, 10), (5, 5, 5), 900, 24, 0, 0.01, 3, (3,), 0.3, 4)
    sequence_case("seq_4mode_l1", (9, 8, 7, 6), (2, 3, 2, 2), 500, 25, 1, 0.05, 3, (2,), 0.2, 5)
    sequence_case("seq_2mode_lf", (30, 25), (4, 3), 300, 26, 0, 0.0, 3, (3,), 0.3, 6)
    sequence_case("seq_5mode_lf", (6, 5, 5, 4, 4), (2, 2, 2, 2, 2), 600, 27, 0, 0.01, 2, (2,), 0.3, 7)
    # a config-1-shaped instance at 1/20 of the entries (BASELINE config 1: 1000^3, R=5)
    sequence_case("seq_c1_scaled", (1000, 1000, 1000), (5, 5, 5), 5000, 1, 0, 0.01, 3, (3,), 0.5, 8)
    sequence_case("seq_c2_shape", (400, 400, 400), (10, 10, 10), 6000, 2, 0, 0.01, 2, (2,), 0.3, 9)
    fit_case()


if __name__ == "__main__":
    main()
