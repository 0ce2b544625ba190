"""Tooling: the data-format row measured -- config-2-sized
COO text (10M entries) written and parsed by vest_io.cpp (all host threads) and
by the reference's own save_coo/load_coo (oracle/_ref), plus the binary cache.
Writes profiles/<tag>_io_bench.json."""
import ctypes as C
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1904_02603_b200 import sparsetuck as st  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
nnz = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
cfg = bench.CONFIG2
coords, vals = bench.synth(cfg["dims"], nnz, cfg["data_seed"])
x = st.SparseTensor(cfg["dims"], coords, vals)
ref = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libsparsetuck_ref.so"))
u64p, u32p, f64p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_double)
out = {"entries": nnz, "threads": os.cpu_count()}
with tempfile.TemporaryDirectory() as d:
    a, b, cbin = os.path.join(d, "ref.coo"), os.path.join(d, "ours.coo"), os.path.join(d, "x.bin")
    t = time.perf_counter()
    st.save_coo(x, b)
    out["save_coo_ours_s"] = time.perf_counter() - t
    dd = np.asarray(x.dims, np.uint64)
    cc = np.ascontiguousarray(x.coords).reshape(-1)
    t = time.perf_counter()
    ref.vr_save_coo(a.encode(), 3, dd.ctypes.data_as(u64p), nnz, cc.ctypes.data_as(u32p),
                    x.values.ctypes.data_as(f64p))
    out["save_coo_ref_s"] = time.perf_counter() - t
    out["bytes"] = os.path.getsize(b)
    out["identical"] = open(a, "rb").read() == open(b, "rb").read()
    t = time.perf_counter()
    y = st.load_coo(b)
    out["load_coo_ours_s"] = time.perf_counter() - t
    order, n = C.c_int(), C.c_uint64()
    t = time.perf_counter()
    ref.vr_load_coo(a.encode(), 0, C.byref(order), C.byref(n), None, None, None)
    out["load_coo_ref_s"] = time.perf_counter() - t
    out["load_equal"] = bool(np.array_equal(y.coords, x.coords) and np.array_equal(y.values, x.values))
    t = time.perf_counter()
    st.save_coo_cache(x, cbin)
    out["cache_save_s"] = time.perf_counter() - t
    t = time.perf_counter()
    z = st.load_coo_cache(cbin)
    out["cache_load_s"] = time.perf_counter() - t
    out["cache_equal"] = bool(np.array_equal(z.values, x.values))
for k in ("save_coo", "load_coo"):
    out[k + "_speedup"] = out[k + "_ref_s"] / out[k + "_ours_s"]
json.dump(out, open(os.path.join(ROOT, "profiles", f"{tag}_io_bench.json"), "w"), indent=1)
print(json.dumps(out))
