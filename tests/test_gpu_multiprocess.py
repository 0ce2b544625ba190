"""The sharded path in real separate processes (one process per rank, as
bench.py runs it under torchrun): two processes on the one B200 of this box,
each driving its own shard context (vest_ctx_create_shard: the rank's
work-balanced rows of every mode) through process-level exchange hooks --
sharded.TorchComm over torch.distributed gloo on the library's CUDA buffers
(host-synchronised collectives; no kernel waits on another process's kernel,
so two ranks can share one GPU).  The replicas must be bit-identical and agree
with a single unsharded context within 1e-9 (rows are independent within a
mode, updates.hpp:153-175; core statistics are sums over entries)."""
import os
import socket
import sys

import numpy as np
import pytest

from parity import assert_close

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    "3mode": dict(dims=[60, 50, 40], ranks=[5, 5, 5], nnz=8000, mask=0.0),
    "4mode_masked": dict(dims=[30, 28, 26, 24], ranks=[8, 8, 8, 8], nnz=8000, mask=0.9),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(case):
    sys.path.insert(0, ROOT)
    from paper_1904_02603_b200 import sparsetuck as st
    c = CASES[case]
    rng = np.random.default_rng(7)
    cells = np.sort(rng.choice(int(np.prod(c["dims"])), c["nnz"], replace=False))
    coords = np.stack(np.unravel_index(cells, c["dims"]), 1).astype(np.uint32)
    x = st.make_tensor(c["dims"], coords, rng.uniform(0, 1, len(cells)))
    m = st.init_random(c["dims"], c["ranks"], 9)
    if c["mask"] > 0:
        cm = (np.random.default_rng(3).random(m.core.shape) < c["mask"]).astype(np.uint8)
        m.core[cm == 1] = 0.0
        m.core_mask = cm
    return x, m, c


def _drive(dev, m):
    dev.set_model(m)
    res = []
    for t in range(4):
        res.append(dev.cd_iteration(0, 0.01))
        if t == 2:
            dev.compute_responsibilities(want=False)
            dev.prune_step(0.2)
    return res, dev.get_model()


def _worker(rank, world, port, case, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1904_02603_b200 import sharded as sh

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    x, m, c = _problem(case)
    dev = sh.ShardDevice(x, c["ranks"], rank, world, sh.TorchComm("cuda"), 0)
    res, mm = _drive(dev, m)
    np.savez(os.path.join(out, f"rank{rank}.npz"), res=np.asarray(res), core=mm.core, core_mask=mm.core_mask,
             local_nnz=np.asarray([dev.local_nnz(n) for n in range(len(c["dims"]))]),
             **{f"f{n}": f for n, f in enumerate(mm.factors)}, **{f"k{n}": k for n, k in enumerate(mm.factor_masks)})
    dev.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_two_processes_one_gpu_match_single_context(case, tmp_path):
    import torch.multiprocessing as mp
    from paper_1904_02603_b200 import sparsetuck as st

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x, m, c = _problem(case)
    dev = st.Device(x, c["ranks"])
    ref_res, ref_m = _drive(dev, m)
    dev.close()
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    N = len(c["dims"])
    # each rank traversed only its rows: the shards' entries partition the tensor
    assert sum(int(o["local_nnz"][N - 1]) for o in outs) == x.nnz()
    for o in outs:
        for a, b in zip(o["res"], ref_res):
            assert abs(a - b) <= 1e-9 * b
        assert_close(o["core"], ref_m.core, "core", tol=1e-9)
        assert np.array_equal(o["core_mask"], ref_m.core_mask)
        for n in range(N):
            assert_close(o[f"f{n}"], ref_m.factors[n], f"factor {n}", tol=1e-9)
            assert np.array_equal(o[f"k{n}"], ref_m.factor_masks[n])
    for key in outs[0].files:  # replicas bit-identical across the processes
        if key != "local_nnz":
            assert np.array_equal(outs[0][key], outs[1][key]), key
