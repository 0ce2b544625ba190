"""CPU-only checks of the product's host side: the C-ABI library loads and
exports every symbol include/vest.h declares (no compute calls without a GPU),
the host utilities (init_random, split, synthetic inputs, sharding plan) match
the reference, and the host control logic (PruneSchedule / StopController /
make_tensor validation) follows pruning.hpp / sparse_tensor.hpp."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

from paper_1904_02603_b200 import _lib
from paper_1904_02603_b200 import sparsetuck as st


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.lib()


def test_library_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "vest.h")).read()
    declared = set(re.findall(r"\b(vest_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 30
    for name in sorted(declared):
        assert hasattr(L, name), f"libvest_cuda.so does not export {name}"
    assert set(_lib.SIGNATURES) >= declared


def test_version_and_counter(L):
    assert b"sm_100a" in L.vest_version()
    assert L.vest_launch_count() == 0  # nothing launched without a device


@pytest.mark.parametrize("f32", ["0", "1"])
@pytest.mark.parametrize("ranks,keep", [([8, 8, 8, 8], 0.1), ([5, 5, 5], 1.0), ([3, 4], 0.5), ([2, 2, 3, 2, 2], 0.3)])
def test_sparse_delta_source_compiles_for_sm100a(L, ranks, keep, f32, monkeypatch):
    """The mask-specialised delta contraction (vest_sparse.cu) and the
    plan-specialised core passes (vest_core_gen.cu) are generated and
    NVRTC-compiled for sm_100a on the host -- no GPU involved -- with fp64 and
    fp32 factor gathers."""
    monkeypatch.setenv("VEST_GATHER_F32", f32)
    g = int(np.prod(ranks))
    mask = (np.random.default_rng(44).random(g) >= keep).astype(np.uint8)
    r = np.asarray(ranks, np.uint64)
    out = np.zeros(1, np.uint64)
    rc = L.vest_sparse_compile_check(len(ranks), _lib.ptr(r, _lib.u64p), _lib.ptr(mask, _lib.u8p),
                                     _lib.ptr(out, _lib.u64p))
    assert rc == 0, L.vest_last_error()
    assert out[0] > 1000  # a cubin


def test_cli_builds_and_reports_usage_errors():
    """tools/sparsetuck_b200 (the reference CLI surface) builds against the C++
    mirror; argument errors fail before any device work."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    exe = os.path.join(ROOT, "tools", "sparsetuck_b200")
    r = subprocess.run([exe, "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "decompose" in r.stdout and "synth" in r.stdout
    for args in (["decompose", "--input", "x.coo"], ["predict", "--model-dir", "d"], ["bogus"],
                 ["decompose", "--input", "x", "--ranks", "2,2", "--reg", "l2"], ["evaluate", "--nope", "1"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True)
        assert r.returncode != 0, args
    r = subprocess.run([exe, "evaluate", "--model-dir", "/nonexistent", "--input", "x"], capture_output=True,
                       text=True)
    assert r.returncode == 1 and r.stderr.startswith("error: ")


def test_init_random_host_matches_reference(L):
    g = golden("init_random")
    for k in range(int(g["ncases"])):
        dims = [int(d) for d in g[f"case{k}_dims"]]
        ranks = [int(r) for r in g[f"case{k}_ranks"]]
        m = st.init_random(dims, ranks, int(g[f"case{k}_seed"]))
        assert np.array_equal(m.core, g[f"case{k}_core"])
        for n in range(len(dims)):
            assert np.array_equal(m.factors[n].reshape(-1), g[f"case{k}_factor{n}"].reshape(-1))


def test_split_matches_reference(L):
    g = golden("split")
    for n in (1200, 1000):
        seed = 5 if n == 1200 else 2024
        x = st.SparseTensor([n], np.arange(n, dtype=np.uint32).reshape(-1, 1), np.arange(n, dtype=np.float64))
        tr, te = st.split_train_test(x, 0.1, seed)
        assert np.array_equal(te.coords[:, 0].astype(np.uint64), g[f"test_{n}"])
        assert np.array_equal(tr.coords[:, 0].astype(np.uint64), g[f"train_{n}"])
    assert (tr.nnz(), te.nnz()) == (900, 100)


def _synth(L, dims, nnz, zipf=None, kind=0, seed=1):
    d = np.asarray(dims, np.uint64)
    z = np.asarray(zipf if zipf else [0.0] * len(dims), np.float64)
    coords = np.zeros(nnz * len(dims), np.uint32)
    vals = np.zeros(nnz)
    rc = L.vest_synth(len(dims), _lib.ptr(d, _lib.u64p), nnz, _lib.ptr(z, _lib.f64p), kind, seed,
                      _lib.ptr(coords, _lib.u32p), _lib.ptr(vals, _lib.f64p))
    assert rc == 0
    return coords.reshape(nnz, len(dims)), vals


def test_synth_distinct_sorted_deterministic(L):
    c1, v1 = _synth(L, [100, 90, 80], 20000)
    c2, v2 = _synth(L, [100, 90, 80], 20000)
    assert np.array_equal(c1, c2) and np.array_equal(v1, v2)
    lin = (c1[:, 0].astype(np.int64) * 90 + c1[:, 1]) * 80 + c1[:, 2]
    assert np.all(np.diff(lin) > 0)  # distinct, row-major order
    assert (c1 < np.array([100, 90, 80])).all()
    assert 0.0 <= v1.min() and v1.max() < 1.0


def test_synth_zipf_and_value_kinds(L):
    c, v = _synth(L, [5000, 3000, 100], 30000, zipf=[1.1, 1.1, 0.0], kind=1)
    counts = np.bincount(c[:, 0], minlength=5000)
    assert counts[0] > 20 * np.median(counts[counts > 0])  # heavy head
    assert set(np.unique(v)) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    c4, v4 = _synth(L, [10 ** 6] * 4, 5000, kind=2)
    assert np.array_equal(v4, v4.astype(np.float32).astype(np.float64))


def test_partition_rows_balanced(L):
    rng = np.random.default_rng(0)
    counts = rng.zipf(1.5, 1000).astype(np.uint64)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    for world in (1, 2, 4, 8):
        b = np.zeros(world + 1, np.uint64)
        assert L.vest_partition_rows(_lib.ptr(off, _lib.u64p), 1000, world, _lib.ptr(b, _lib.u64p)) == 0
        assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b.astype(np.int64)) >= 0)
        loads = off[b[1:]] - off[b[:-1]]
        assert loads.sum() == off[-1]
        # every boundary is the first row reaching its share
        for r in range(1, world):
            target = int(off[-1]) * r // world
            assert off[b[r]] >= target and (b[r] == b[r - 1] or off[b[r] - 1] < target)


def test_sharded_partition_row_cost():
    """sharded.partition balances entries + row_cost per non-empty row: a Zipf
    mode's long tail of short rows moves its boundary towards the tail."""
    from paper_1904_02603_b200 import sharded as sh
    rng = np.random.default_rng(3)
    rows = np.minimum(rng.zipf(1.3, 20000), 2000).astype(np.int64) - 1
    rows = rows[rows < 2000]
    coords = np.stack([rows, rng.integers(0, 50, len(rows)), rng.integers(0, 40, len(rows))], 1)
    x = st.SparseTensor([2000, 50, 40], coords.astype(np.uint32), np.ones(len(rows)))
    for rc in (0, 8):
        b = sh.partition(x, 4, row_cost=rc)[0].astype(np.int64)
        counts = np.bincount(rows, minlength=2000)
        w = counts + rc * (counts > 0)
        loads = [w[b[r]:b[r + 1]].sum() for r in range(4)]
        assert b[0] == 0 and b[-1] == 2000 and np.all(np.diff(b) >= 0)
        assert max(loads) <= w.sum() / 4 + w.max()  # balanced up to one row
    b0, b8 = sh.partition(x, 4, row_cost=0)[0], sh.partition(x, 4, row_cost=8)[0]
    assert b8[-2] >= b0[-2]  # the tail rank owns fewer (costlier) short rows


# ---- host control logic (pruning.hpp:17-81), cases from tests/test_pruning.cpp:17-92
def test_prune_schedule():
    s = st.PruneSchedule(0.01, 0.1)
    assert s.rate(1) == pytest.approx(0.01)
    assert s.rate(5) == pytest.approx(0.05)
    assert s.rate(20) == 0.1
    with pytest.raises(ValueError):
        s.rate(0)
    for bad in ((0.0, 0.1), (0.2, 0.1), (0.1, 1.0)):
        with pytest.raises(ValueError):
            st.PruneSchedule(*bad).validate()


def test_stop_controller_manual_latches():
    c = st.StopController(st.StopMode.Manual, 0.3)
    assert c.should_prune(0.1, 0.5, 0.01)
    assert not c.should_prune(0.3, 0.5, 0.01)
    assert c.stopped()
    assert not c.should_prune(0.0, 0.5, 0.01)


def test_stop_controller_auto_elbow():
    c = st.StopController(st.StopMode.Auto, 0.0, 0.05)
    for re in (0.10, 0.11):
        assert c.should_prune(0.0, re, 0.01)
        c.record_prune_event(re)
    # (0.14 + 0.10 - 2 * 0.11) / 0.01 = 2.0 > 0.05 -> stop and latch
    assert not c.should_prune(0.0, 0.14, 0.01)
    assert c.stopped() and not c.should_prune(0.0, 0.1, 0.01)
    flat = st.StopController(st.StopMode.Auto)
    for _ in range(20):
        assert flat.should_prune(0.0, 0.1, 0.05)
        flat.record_prune_event(0.1)
    z = st.StopController(st.StopMode.Manual, 0.5)
    assert not z.should_prune(0.0, 0.0, 0.1) and not z.stopped()  # perfect fit: no latch


def test_make_tensor_validation():
    with pytest.raises(ValueError, match="order must be at least 1"):
        st.make_tensor([], [], [])
    with pytest.raises(ValueError, match="dimensions must be positive"):
        st.make_tensor([3, 0], [], [])
    with pytest.raises(ValueError, match="does not match"):
        st.make_tensor([3, 3], [0, 1, 2], [1.0, 2.0])
    with pytest.raises(ValueError, match="out of bounds"):
        st.make_tensor([3, 3], [[0, 3]], [1.0])
    with pytest.raises(ValueError, match="duplicate"):
        st.make_tensor([3, 3], [[1, 2], [0, 0], [1, 2]], [1.0, 2.0, 3.0])
    x = st.make_tensor([3, 4], [[0, 0], [1, 1]], [3.0, 4.0])
    assert x.frobenius_norm() == 5.0  # tests/test_sparse_tensor.cpp:38-41


def test_fit_config_validation():
    x = st.make_tensor([3, 4], [[0, 0], [1, 1]], [3.0, 4.0])
    for kw, msg in (({"ranks": [1]}, "ranks order"), ({"ranks": [1, 0]}, "ranks must be positive"),
                    ({"ranks": [1, 1], "lam": -1.0}, "lambda"), ({"ranks": [1, 1], "tol": -1.0}, "tol"),
                    ({"ranks": [1, 1], "max_iters": 0}, "max_iters"),
                    ({"ranks": [1, 1], "target_sparsity": 1.0}, "target sparsity")):
        with pytest.raises(ValueError, match=msg):
            st.fit(x, st.TrainConfig(**kw))
    z = st.make_tensor([3, 4], [[0, 0]], [0.0])
    with pytest.raises(ValueError, match="all zero"):
        st.fit(z, st.TrainConfig(ranks=[1, 1]))
