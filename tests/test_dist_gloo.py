"""The multi-rank path on CPU: world_size 2, torch.distributed gloo.

* the communication hooks (paper_1904_02603_b200.sharded.TorchComm) on host
  buffers: allreduce_sum and allgather_rows semantics;
* the sharded CD algebra the CUDA path implements: each rank
  updates only its nnz-balanced rows of each mode and the rows are exchanged
  with allgather_rows -> identical (bit-for-bit) to the single-process
  update_all_factors of the oracle; the core sweep's block statistics are
  rank-partial sums over the rank's last-mode slices, all-reduced, and every
  rank runs the same sequential block solve -> equal to the oracle's
  update_core within 1e-9.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance():
    rng = np.random.default_rng(5)
    dims, ranks = [30, 24, 20], [3, 3, 2]
    cells = np.sort(rng.choice(int(np.prod(dims)), 1500, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    return dims, ranks, coords, rng.uniform(0, 1, len(cells))


def _blocked_core_sweep(O, s, dims, ranks, coords, values, lam, comm, lo2, hi2):
    """Fiber-blocked exact Gauss-Seidel core sweep with rank-partial statistics
    (the algebra of vest_core.cu, restated densely in numpy)."""
    core, cm, fs, ms = s.get_model()
    r_full, _, _, _ = s.compute_residuals(1)
    own = (coords[:, 2] >= lo2) & (coords[:, 2] < hi2)
    cz, r = coords[own], r_full[own].copy()
    J0, J1, J2 = ranks
    for b0 in range(J0):  # block = the fibers of prefix beta_0 = b0
        w = fs[0][cz[:, 0], b0]
        P = (w[:, None, None] * fs[1][cz[:, 1], :][:, :, None] * fs[2][cz[:, 2], :][:, None, :]).reshape(len(cz), -1)
        H = np.ascontiguousarray(P.T @ P)
        c = np.ascontiguousarray(P.T @ r)
        comm.allreduce(H.ctypes.data_as(C.POINTER(C.c_double)), H.size, 0)
        comm.allreduce(c.ctypes.data_as(C.POINTER(C.c_double)), c.size, 0)
        dg = np.zeros(J1 * J2)
        for q in range(J1 * J2):
            lin = b0 * J1 * J2 + q
            if cm[lin]:
                continue
            num = c[q] - H[q, :q] @ dg[:q] + core[lin] * H[q, q]
            den = H[q, q]
            if den + lam != 0.0:
                g_new = num / (den + lam)
                dg[q] = g_new - core[lin]
                core[lin] = g_new
        r -= P @ dg
    return core


def _worker(rank, world, port, q):
    try:
        import sys

        sys.path.insert(0, ROOT)
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as O
        from paper_1904_02603_b200 import sharded as sh
        from paper_1904_02603_b200 import sparsetuck as st

        comm = sh.TorchComm(device="cpu")
        # 1. allreduce_sum on a host buffer
        buf = np.full(7, float(rank + 1))
        comm.allreduce(buf.ctypes.data_as(C.POINTER(C.c_double)), 7, 0)
        assert np.all(buf == sum(range(1, world + 1)))
        # 2. allgather_rows: rank r owns rows [b[r], b[r+1]) of a 10 x 3 buffer
        class Fake:
            pass
        fake = Fake()
        fake.world = world
        fake.bounds = [np.array([0, 4, 10], np.uint64)]
        rows = np.zeros((10, 3))
        b = fake.bounds[0]
        rows[int(b[rank]):int(b[rank + 1])] = rank + 1
        comm.allgather_rows(fake, 0, rows.ctypes.data_as(C.POINTER(C.c_double)), 3, 0)
        assert np.all(rows[:4] == 1) and np.all(rows[4:] == 2)
        # 3. sharded factor sweep == oracle update_all_factors, bit-for-bit
        dims, ranks, coords, values = _instance()
        x = st.SparseTensor(dims, coords, values)
        bounds = sh.partition(x, world)
        s = O.Session(dims, coords, values, ranks, "port")
        s.init_random(3)
        ref = O.Session(dims, coords, values, ranks, "port")
        ref.init_random(3)
        ref.update_all_factors(0, 0.05, 1)
        for n in range(3):
            lo, hi = int(bounds[n][rank]), int(bounds[n][rank + 1])
            for i in range(lo, hi):
                s.update_factor_row(0, n, i, 0.05)
            core, cm, fs, ms = s.get_model()
            f = np.ascontiguousarray(fs[n])
            comm.allgather_rows(type("B", (), {"world": world, "bounds": bounds})(), n,
                                f.ctypes.data_as(C.POINTER(C.c_double)), ranks[n], 0)
            fs[n] = f
            s.set_model(core, cm, fs, ms)
        _, _, fs, _ = s.get_model()
        _, _, fr, _ = ref.get_model()
        for n in range(3):
            assert np.array_equal(fs[n], fr[n]), f"factor {n} differs"
        # 4. sharded blocked core sweep == oracle update_core
        core = _blocked_core_sweep(O, s, dims, ranks, coords, values, 0.05, comm,
                                   int(bounds[2][rank]), int(bounds[2][rank + 1]))
        ref.update_core(0, 0.05, 1)
        core_ref = ref.get_model()[0]
        err = np.abs(core - core_ref).max() / np.abs(core_ref).max()
        assert err <= 1e-9, err
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        import traceback

        q.put((rank, "".join(traceback.format_exception(e))))


def test_gloo_world2_sharded_path(oracle_lib):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
