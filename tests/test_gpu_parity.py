"""GPU parity: the CUDA path (through the C-ABI, via the Python mirror) against
the reference's own outputs (tests/golden, made by the unmodified reference
headers) and against the C restatement (oracle/) on seeded random instances.

Protocol (SURVEY.md 7 "parity logistics"): phase-wise.  Before every phase the
device model is re-synced to the reference's state, so each kernel is checked
on exactly the reference's input; tolerances are in tests/parity.py.
"""
import numpy as np
import pytest

from conftest import SEQ_CASES, golden
from parity import assert_close, assert_masks, assert_resp

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")


def _tensor(g):
    return st.SparseTensor([int(d) for d in g["dims"]], g["coords"].astype(np.uint32), g["values"])


def _model(g, dims, ranks, core, cm, fs, ms):
    return st.TuckerModel(list(dims), list(ranks), core.copy(), cm.copy(), [f.copy() for f in fs],
                          [m.copy() for m in ms])


def run_golden_phases(case, generic=False):
    g = golden(case)
    dims = [int(d) for d in g["dims"]]
    ranks = [int(r) for r in g["ranks"]]
    N = len(dims)
    x = _tensor(g)
    dev = st.Device(x, ranks)
    if generic:
        dev.force_generic(True)
    # device CSF == reference ModeIndex, bit for bit
    for n in range(N):
        off, ids = dev.mode_index(n)
        assert np.array_equal(off, g[f"index_offsets{n}"])
        assert np.array_equal(ids, g[f"index_ids{n}"])
    core, cm = g["init_core"], g["init_core_mask"]
    fs = [g[f"init_factor{n}"] for n in range(N)]
    ms = [g[f"init_fmask{n}"] for n in range(N)]
    reg, lam = int(g["reg"]), float(g["lam"])
    prune_at = set(int(t) for t in g["prune_at"])
    for t in range(1, int(g["iters"]) + 1):
        dev.set_model(_model(g, dims, ranks, core, cm, fs, ms))
        dev.update_all_factors(reg, lam)
        m = dev.get_model()
        for n in range(N):
            assert_close(m.factors[n], g[f"t{t}_factors_factor{n}"], f"{case} t{t} factor{n}")
            assert np.all(m.factors[n][ms[n] == 1] == 0.0), "masked factor written"
        fs = [g[f"t{t}_factors_factor{n}"] for n in range(N)]
        dev.set_model(_model(g, dims, ranks, core, cm, fs, ms))
        dev.update_core(reg, lam)
        m = dev.get_model()
        assert_close(m.core, g[f"t{t}_core"], f"{case} t{t} core")
        assert np.all(m.core[cm == 1] == 0.0), "masked core written"
        core = g[f"t{t}_core"]
        dev.set_model(_model(g, dims, ranks, core, cm, fs, ms))
        res = dev.compute_residuals(want_r=True)
        assert_close(res.r, g[f"t{t}_r"], f"{case} t{t} r")
        assert abs(res.re - g[f"t{t}_re"]) <= 1e-6 * abs(g[f"t{t}_re"]), (res.re, g[f"t{t}_re"])
        assert res.x_norm == g[f"t{t}_x_norm"]
        zero, _ = dev.sparsity()
        assert zero == g[f"t{t}_sparsity"]
        if t in prune_at:
            tab = dev.compute_responsibilities()
            assert_resp(tab.core, g[f"t{t}_resp_core"], f"{case} t{t} resp core")
            for n in range(N):
                assert_resp(tab.factors[n], g[f"t{t}_resp_factor{n}"], f"{case} t{t} resp factor{n}")
            counts = dev.prune_step(float(g["pr"]))
            ref_counts = g[f"t{t}_prune_counts"]
            assert [counts.core] + counts.factors == [int(c) for c in ref_counts]
            m = dev.get_model()
            assert_masks(m.core_mask, g[f"t{t}_pruned_core_mask"], g[f"t{t}_resp_core"], cm, "core mask")
            for n in range(N):
                assert_masks(m.factor_masks[n], g[f"t{t}_pruned_fmask{n}"], g[f"t{t}_resp_factor{n}"], ms[n],
                             f"factor{n} mask")
            core = g[f"t{t}_pruned_core"]
            cm = g[f"t{t}_pruned_core_mask"]
            fs = [g[f"t{t}_pruned_factor{n}"] for n in range(N)]
            ms = [g[f"t{t}_pruned_fmask{n}"] for n in range(N)]
    # normalisation of the final (reference) state
    dev.set_model(_model(g, dims, ranks, core, cm, fs, ms))
    dev.normalize_columns()
    m = dev.get_model()
    assert_close(m.core, g["normalized_core"], f"{case} normalized core")
    for n in range(N):
        assert_close(m.factors[n], g[f"normalized_factor{n}"], f"{case} normalized factor{n}")
    # probes: delta (reference cell order -> bit-identical) and predict
    dev.set_model(_model(g, dims, ranks, g["normalized_core"], cm, [g[f"normalized_factor{n}"] for n in range(N)], ms))
    probe = g["probe_coords"]
    got = dev.predict(probe)
    assert_close(got, g["probe_recon"], "predict")
    for n in range(N):
        d = np.stack([dev.compute_delta(c, n) for c in probe])
        assert np.array_equal(d, g[f"probe_delta{n}"])
    dev.close()


@pytest.mark.parametrize("case", SEQ_CASES)
def test_golden_phases(case):
    run_golden_phases(case)


@pytest.mark.parametrize("case", ["seq_c1_scaled", "seq_c2_shape"])
def test_golden_phases_generic_kernels(case):
    """The same fixtures through the generic (runtime-rank) kernels."""
    run_golden_phases(case, generic=True)


def test_specialised_path_selected():
    g = golden("seq_c2_shape")
    dev = st.Device(_tensor(g), [10, 10, 10])
    assert dev.specialised()
    g = golden("seq_543_lf")
    dev2 = st.Device(_tensor(g), [2, 3, 2])
    assert not dev2.specialised()


def test_init_random_matches_reference():
    g = golden("init_random")
    for k in range(int(g["ncases"])):
        dims = [int(d) for d in g[f"case{k}_dims"]]
        ranks = [int(r) for r in g[f"case{k}_ranks"]]
        m = st.init_random(dims, ranks, int(g[f"case{k}_seed"]))
        assert np.array_equal(m.core, g[f"case{k}_core"])
        for n in range(len(dims)):
            assert np.array_equal(m.factors[n].reshape(-1), g[f"case{k}_factor{n}"].reshape(-1))
        x = st.SparseTensor(dims, np.zeros((1, len(dims)), np.uint32), np.ones(1))
        dev = st.Device(x, ranks)
        dev.init_random(int(g[f"case{k}_seed"]))
        md = dev.get_model()
        assert np.array_equal(md.core, g[f"case{k}_core"])


@pytest.mark.parametrize("dims,nnz", [([70000, 300, 5], 1_500_001), ([3, 1 << 20], 400_000), ([40, 30, 20], 8193)])
def test_mode_index_radix_sort_vs_stable_argsort(dims, nnz):
    """K1 (vest_sort.cu, the hand-written stable LSD radix sort behind the CSF
    build): per-mode index == a stable argsort of each coordinate
    (sparse_tensor.hpp:119-137: ids ascending within a slice), over 1-3 radix
    passes per mode, a partial last tile, a Zipf-skewed mode and a 20-bit mode;
    a duplicate coordinate is still detected through the sorted order."""
    rng = np.random.default_rng(17)
    total = int(np.prod([float(d) for d in dims]))
    nnz = min(nnz, total // 2)
    # distinct coordinates: distinct linear ids, skewed towards low indices of mode 0
    lin = np.unique((rng.random(2 * nnz) ** 2 * total).astype(np.int64))[:nnz]
    rng.shuffle(lin)
    coords = np.stack(np.unravel_index(lin, dims), 1).astype(np.uint32)
    vals = rng.random(len(lin))
    x = st.SparseTensor(list(dims), coords, vals)
    dev = st.Device(x, [2] * len(dims))
    for n in range(len(dims)):
        off, ids = dev.mode_index(n)
        want = np.argsort(coords[:, n], kind="stable")
        assert np.array_equal(ids, want.astype(ids.dtype))
        cnt = np.bincount(coords[:, n], minlength=dims[n])
        assert np.array_equal(off, np.concatenate([[0], np.cumsum(cnt)]).astype(off.dtype))
    dev.close()
    bad = coords.copy()
    bad[-1] = bad[len(bad) // 3]
    with pytest.raises(ValueError, match="duplicate coordinate"):
        st.make_tensor(list(dims), bad, vals)
