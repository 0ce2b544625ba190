"""Workload for compute-sanitizer (memcheck / racecheck / synccheck), one tool
per run (profiles/run_sanitizers.sh): small instances that still reach every
kernel family -- 3-mode rank-specialised sweep (cp.async staging, DMMA Gram,
bulk copies, last-CTA reductions, iteration graph replay), short rows and heavy
split rows, a 4-mode 90%-masked core through the NVRTC kernels (fused factor
update, mask-specialised delta, plan-specialised core passes, sampled Gram,
fp32 gathers), a dense 5-mode core, responsibilities, prune, predict."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1904_02603_b200 import sparsetuck as st  # noqa: E402
from test_gpu_oracle import random_instance  # noqa: E402


def run(dims, ranks, nnz, seed, iters, mask=0.0, skew=None, sparse=None, gen=None, f32=False, fused=None):
    coords, values, m = random_instance(dims, ranks, nnz, seed, mask_frac=mask, skew=skew)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    if sparse is not None:
        dev.set_sparse_delta(sparse)
    if gen is not None:
        dev.set_core_gen(gen)
    if fused is not None:
        dev.set_sparse_fused(fused)
    dev.set_gather_f32(f32)
    dev.set_model(m)
    res = [dev.cd_iteration(0, 0.01) for _ in range(iters)]
    dev.compute_responsibilities(want=False)
    dev.prune_step(0.2)
    res.append(dev.cd_iteration(1, 0.05))
    dev.predict(coords[:100])
    dev.close()
    print(dims, ranks, [round(r, 6) for r in res], flush=True)


run([200, 150, 100], [5, 5, 5], 6000, 1, 6)                         # graph capture + replay from iteration 5
run([80, 70, 60], [10, 10, 10], 6000, 2, 2)
run([3, 60, 60], [5, 5, 5], 9000, 3, 2, skew=None)                   # heavy rows split across chunks
run([12, 40, 30], [5, 5, 5], 8000, 4, 2, skew=1.6)                   # skewed: short rows lane-per-row
run([20, 18, 16, 14], [8, 8, 8, 8], 5000, 5, 2, mask=0.9, sparse=1, gen=1)             # fused + generated
run([20, 18, 16, 14], [8, 8, 8, 8], 5000, 6, 2, mask=0.9, sparse=1, gen=1, fused=0)    # delta through HBM
run([20, 18, 16, 14], [8, 8, 8, 8], 5000, 7, 2, mask=0.9, sparse=1, gen=1, f32=True)  # fp32 gathers
run([9, 8, 8, 7, 7], [5, 5, 5, 5, 5], 4000, 8, 2, gen=1)
print("sanitize workload done")
