"""The sharded (multi-GPU) path on one GPU: W shard contexts, each owning an
nnz-balanced row range of every mode, exchange through the library's
communication hooks (paper_1904_02603_b200.sharded.LocalGroup emulates the ranks
as threads of one process; every exchange is host-synchronised, no kernel waits
on another).  The result must equal the single-context run up to summation order,
and all replicas must stay bit-identical."""
import numpy as np
import pytest

from parity import assert_close

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")
sh = pytest.importorskip("paper_1904_02603_b200.sharded")


def _instance(dims, ranks, nnz, seed, zipf=False):
    rng = np.random.default_rng(seed)
    total = int(np.prod(dims))
    if zipf:
        w = 1.0 / np.arange(1, dims[0] + 1) ** 1.2
        rows = rng.choice(dims[0], size=nnz * 3, p=w / w.sum())
        rest = rng.integers(0, total // dims[0], size=nnz * 3)
        cells = np.unique(rows.astype(np.int64) * (total // dims[0]) + rest)[:nnz]
        cells = np.sort(cells)
    else:
        cells = np.sort(rng.choice(total, size=nnz, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    return st.make_tensor(dims, coords, rng.uniform(0.0, 1.0, len(cells)))


def _run_single(x, ranks, iters, seed, pr):
    dev = st.Device(x, ranks)
    dev.init_random(seed)
    res = []
    for t in range(iters):
        res.append(dev.cd_iteration(0, 0.01))
        if pr and t == iters - 2:
            dev.compute_responsibilities(want=False)
            dev.prune_step(pr)
    return res, dev.get_model()


def _run_sharded(x, ranks, iters, seed, pr, world):
    group = sh.LocalGroup(world)
    bounds = sh.partition(x, world)
    devs = [sh.ShardDevice(x, ranks, r, world, group.hooks_for(r), bounds=bounds) for r in range(world)]

    def body(r):
        d = devs[r]
        d.init_random(seed)
        res = []
        for t in range(iters):
            res.append(d.cd_iteration(0, 0.01))
            if pr and t == iters - 2:
                d.compute_responsibilities(want=False)
                d.prune_step(pr)
        return res, d.get_model()

    return group.run([lambda r=r: body(r) for r in range(world)]), devs


@pytest.mark.parametrize("ranks", [[5, 5, 5], [10, 10, 10], [3, 2, 2]])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_matches_single(ranks, world):
    x = _instance([60, 50, 40], ranks, 8000, 1)
    ref_res, ref_m = _run_single(x, ranks, 4, 7, 0.2)
    outs, devs = _run_sharded(x, ranks, 4, 7, 0.2, world)
    assert sum(d.local_nnz(0) for d in devs) == x.nnz()
    for res, m in outs:
        for a, b in zip(res, ref_res):
            assert abs(a - b) <= 1e-9 * b
        assert_close(m.core, ref_m.core, "sharded core", tol=1e-9)
        for n in range(3):
            assert_close(m.factors[n], ref_m.factors[n], f"sharded factor{n}", tol=1e-9)
            assert np.array_equal(m.factor_masks[n], ref_m.factor_masks[n])
    # replicas bit-identical across ranks
    m0 = outs[0][1]
    for _, m in outs[1:]:
        assert np.array_equal(m.core, m0.core)
        for n in range(3):
            assert np.array_equal(m.factors[n], m0.factors[n])


def test_sharded_skewed_rows():
    x = _instance([40, 60, 50], [5, 5, 5], 9000, 2, zipf=True)
    ref_res, ref_m = _run_single(x, [5, 5, 5], 3, 3, 0.0)
    outs, devs = _run_sharded(x, [5, 5, 5], 3, 3, 0.0, 2)
    for res, m in outs:
        for a, b in zip(res, ref_res):
            assert abs(a - b) <= 1e-9 * b
        assert_close(m.core, ref_m.core, "core", tol=1e-9)


# 4- and 5-mode shapes: the general core sweep with plan-specialised passes and,
# for the 90 %-masked core, the mask-specialised delta (both NVRTC-compiled),
# through the shard exchange points
@pytest.mark.parametrize("dims,ranks,mf", [([30, 28, 26, 24], [8, 8, 8, 8], 0.9), ([9, 9, 8, 8, 7], [5, 5, 5, 5, 5], 0.0)])
def test_sharded_generated_kernels(dims, ranks, mf):
    x = _instance(dims, ranks, 8000, 5)
    m = st.init_random(dims, ranks, 9)
    if mf > 0:
        cm = (np.random.default_rng(3).random(m.core.shape) < mf).astype(np.uint8)
        m.core[cm == 1] = 0.0
        m.core_mask = cm
    dev = st.Device(x, ranks)
    dev.set_model(m)
    assert dev.sparse_delta_active() == (mf > 0)
    ref_res = [dev.cd_iteration(0, 0.01) for _ in range(3)]
    ref_m = dev.get_model()
    group = sh.LocalGroup(2)
    bounds = sh.partition(x, 2)
    devs = [sh.ShardDevice(x, ranks, r, 2, group.hooks_for(r), bounds=bounds) for r in range(2)]

    def body(r):
        devs[r].set_model(m)
        return [devs[r].cd_iteration(0, 0.01) for _ in range(3)], devs[r].get_model()

    outs = group.run([lambda r=r: body(r) for r in range(2)])
    for res, mm in outs:
        for a, b in zip(res, ref_res):
            assert abs(a - b) <= 1e-9 * b
        assert_close(mm.core, ref_m.core, "core", tol=1e-9)
        for n in range(len(dims)):
            assert_close(mm.factors[n], ref_m.factors[n], f"factor{n}", tol=1e-9)
    assert np.array_equal(outs[0][1].core, outs[1][1].core)
