"""Golden outputs of the reference's planted-model generator (gen_synthetic,
synthetic.hpp:105-155) for the CLI's `synth` command, produced by the
unmodified reference headers through oracle/_ref (oracle/ref_shim.cpp
vr_gen_synthetic).  Run in the build container:

    make -C oracle && python tests/golden/make_synth_golden.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libsparsetuck_ref.so"))

SPECS = {  # name: dims, ranks, nnz, density, noise, seed
    "synth_sparse": ([40, 30, 20], [3, 4, 2], 2000, 0.7, 0.05, 11),  # rejection-sampled coordinates
    "synth_dense": ([6, 5, 4], [2, 2, 3], 90, 1.0, 0.0, 5),          # partial Fisher-Yates regime
}


def ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


for name, (dims, ranks, nnz, density, noise, seed) in SPECS.items():
    N = len(dims)
    d = np.asarray(dims, np.uint64)
    r = np.asarray(ranks, np.uint64)
    coords = np.zeros(nnz * N, np.uint32)
    values = np.zeros(nnz)
    core = np.zeros(int(np.prod(ranks)))
    cm = np.zeros(int(np.prod(ranks)), np.uint8)
    fs = [np.zeros(a * b) for a, b in zip(dims, ranks)]
    ms = [np.zeros(a * b, np.uint8) for a, b in zip(dims, ranks)]
    fp = (C.POINTER(C.c_double) * N)(*[ptr(f, C.c_double) for f in fs])
    mp = (C.POINTER(C.c_uint8) * N)(*[ptr(m, C.c_uint8) for m in ms])
    rc = L.vr_gen_synthetic(N, ptr(d, C.c_uint64), ptr(r, C.c_uint64), C.c_uint64(nnz), C.c_double(density),
                            C.c_double(noise), C.c_uint64(seed), ptr(coords, C.c_uint32), ptr(values, C.c_double),
                            ptr(core, C.c_double), ptr(cm, C.c_uint8), fp, mp)
    assert rc == 0, L.vr_last_error
    out = dict(dims=d, ranks=r, nnz=np.uint64(nnz), density=density, noise=noise, seed=np.uint64(seed),
               coords=coords.reshape(nnz, N), values=values, core=core, core_mask=cm)
    for n in range(N):
        out[f"factor{n}"] = fs[n]
        out[f"fmask{n}"] = ms[n]
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")
