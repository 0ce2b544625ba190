"""Tooling: time the reference-facing e2e step's parts (set_model / cd_iteration /
get_model with pinned host buffers) on config 2."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1904_02603_b200 import sparsetuck as st  # noqa: E402

cfg = bench.CONFIG2
coords, vals = bench.synth(cfg["dims"], cfg["nnz"], cfg["data_seed"])
dev = st.Device(st.SparseTensor(cfg["dims"], coords, vals), cfg["ranks"], 0)
dev.init_random(cfg["seed"])
for _ in range(3):
    dev.cd_iteration(0, 0.01)
m = dev.get_model()


def pin(a):
    t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.uint8: torch.uint8}[a.dtype.type], pin_memory=True)
    t.numpy()[...] = a
    pin.keep.append(t)
    return t.numpy()


pin.keep = []
m = st.TuckerModel(m.dims, m.ranks, pin(m.core), pin(m.core_mask), [pin(f) for f in m.factors],
                   [pin(k) for k in m.factor_masks])
for rep in range(4):
    t0 = time.perf_counter()
    dev.set_model(m)
    t1 = time.perf_counter()
    dev.cd_iteration(0, 0.01)
    t2 = time.perf_counter()
    dev.get_model(into=m)
    t3 = time.perf_counter()
    dev.cd_iteration(0, 0.01)
    t4 = time.perf_counter()
    print(f"set {1e3*(t1-t0):.2f} ms  iter-after-set {1e3*(t2-t1):.2f} ms  get {1e3*(t3-t2):.2f} ms  "
          f"plain iter {1e3*(t4-t3):.2f} ms")
