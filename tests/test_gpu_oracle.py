"""GPU path vs the C restatement (oracle/vest_oracle.c, pinned bit-exact to the
reference by tests/test_oracle.py) on seeded random instances that cover the
edge cases the reference's suite tests: masked positions, L1 and LF, empty
rows, rows heavier than one work chunk (split-row reduction), 2..5 modes,
generic and rank-specialised kernels, zero-denominator policies, the fully
pruned fixed point, perfect fits and prune ties."""
import numpy as np
import pytest

from parity import assert_close, assert_masks, assert_resp

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")
from oracle import oracle as O  # noqa: E402  (test infrastructure only)


def random_instance(dims, ranks, nnz, seed, mask_frac=0.0, lo=-1.0, hi=2.0, skew=None):
    rng = np.random.default_rng(seed)
    total = int(np.prod(dims))
    if skew is None:
        cells = np.sort(rng.choice(total, size=nnz, replace=False))
    else:
        # skewed rows on mode 0: geometric-ish row weights
        w = np.concatenate([np.full(int(np.prod(dims[1:])), skew ** (-i)) for i in range(dims[0])])
        w /= w.sum()
        cells = np.sort(rng.choice(total, size=nnz, replace=False, p=w))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    values = rng.uniform(lo, hi, nnz)
    m = st.init_random(dims, ranks, int(rng.integers(1 << 30)))
    if mask_frac > 0:
        cmk = (rng.random(m.core.shape) < mask_frac).astype(np.uint8)
        m.core[cmk == 1] = 0.0
        m.core_mask = cmk
        for n in range(len(dims)):
            fm = (rng.random(m.factors[n].shape) < mask_frac).astype(np.uint8)
            m.factors[n][fm == 1] = 0.0
            m.factor_masks[n] = fm
    return coords, values, m


def oracle_session(dims, ranks, coords, values, m):
    s = O.Session(dims, coords, values, ranks, "port")
    s.set_model(m.core, m.core_mask, m.factors, m.factor_masks)
    return s


def model_of(s, dims, ranks):
    core, cm, fs, ms = s.get_model()
    return st.TuckerModel(list(dims), list(ranks), core, cm, fs, ms)


def phases(dims, ranks, nnz, seed, reg, lam, iters=2, pr=0.3, generic=False, sparse=None, core_gen=None, **kw):
    coords, values, m = random_instance(dims, ranks, nnz, seed, **kw)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    if generic:
        dev.force_generic(True)
    if core_gen is not None:
        dev.set_core_gen(core_gen)
    if sparse is not None:
        dev.set_sparse_delta(sparse)
        assert dev.sparse_delta_active() == bool(sparse)
    s = oracle_session(dims, ranks, coords, values, m)
    N = len(dims)
    for t in range(iters):
        ref = model_of(s, dims, ranks)
        dev.set_model(ref)
        dev.update_all_factors(reg, lam)
        s.update_all_factors(reg, lam, 1)
        got, want = dev.get_model(), model_of(s, dims, ranks)
        for n in range(N):
            assert_close(got.factors[n], want.factors[n], f"factor{n} t{t}")
            assert np.all(got.factors[n][want.factor_masks[n] == 1] == 0.0)
        dev.set_model(want)
        dev.update_core(reg, lam)
        s.update_core(reg, lam, 1)
        got, want = dev.get_model(), model_of(s, dims, ranks)
        assert_close(got.core, want.core, f"core t{t}")
        dev.set_model(want)
        res = dev.compute_residuals(want_r=True)
        r_ref, ss, xn, re = s.compute_residuals(1)
        assert_close(res.r, r_ref, "residual")
        assert abs(res.re - re) <= 1e-6 * re
        tab = dev.compute_responsibilities()
        rc, rf = s.compute_responsibilities(1)
        assert_resp(tab.core, rc, "resp core")
        for n in range(N):
            assert_resp(tab.factors[n], rf[n], f"resp factor{n}")
        counts = dev.prune_step(pr)
        ref_counts = s.prune_step(pr)
        assert [counts.core] + counts.factors == [int(c) for c in ref_counts]
        got, want = dev.get_model(), model_of(s, dims, ranks)
        assert_masks(got.core_mask, want.core_mask, rc, ref.core_mask, "core mask")
        for n in range(N):
            assert_masks(got.factor_masks[n], want.factor_masks[n], rf[n], ref.factor_masks[n], f"fmask{n}")
    dev.close()


@pytest.mark.parametrize("reg,lam", [(0, 0.01), (0, 0.0), (1, 0.05), (1, 0.7)])
@pytest.mark.parametrize("generic", [False, True])
def test_config1_ranks(reg, lam, generic):
    phases([60, 50, 40], [5, 5, 5], 3000, 11, reg, lam, generic=generic, mask_frac=0.1)


@pytest.mark.parametrize("ranks", [[10, 10, 10], [10, 10, 5]])
def test_config23_ranks(ranks):
    phases([80, 70, 60], ranks, 6000, 12, 0, 0.01, mask_frac=0.05)
    phases([80, 70, 60], ranks, 6000, 13, 1, 0.1)


def test_config4_ranks_sparse_core():
    phases([20, 18, 16, 14], [8, 8, 8, 8], 5000, 14, 0, 0.01, iters=1, mask_frac=0.9)
    phases([20, 18, 16, 14], [8, 8, 8, 8], 5000, 14, 0, 0.01, iters=1, mask_frac=0.9, sparse=0)


def test_sparse_delta_auto_selection():
    coords, values, m = random_instance([20, 18, 16, 14], [8, 8, 8, 8], 3000, 3, mask_frac=0.9)
    dev = st.Device(st.make_tensor([20, 18, 16, 14], coords, values), [8, 8, 8, 8])
    dev.set_model(m)
    assert dev.sparse_delta_active()  # 10 %-dense core: mask-specialised contraction
    coords, values, m = random_instance([20, 18, 16], [8, 8, 8], 3000, 3)
    dev = st.Device(st.make_tensor([20, 18, 16], coords, values), [8, 8, 8])
    dev.set_model(m)
    assert not dev.sparse_delta_active()  # dense core: factorised kernels


# the mask-specialised (NVRTC) contraction forced on: every order, L1/LF,
# masks, heavy split rows; recompiled when a prune changes the mask
@pytest.mark.parametrize("dims,ranks,mf", [([20, 18, 16, 14], [8, 8, 8, 8], 0.9), ([60, 50, 40], [5, 5, 5], 0.3),
                                           ([30, 25], [4, 3], 0.2), ([7, 6, 5, 4, 3], [2, 2, 3, 2, 2], 0.2),
                                           ([9, 8, 8, 7, 7], [5, 5, 5, 5, 5], 0.5)])
@pytest.mark.parametrize("reg,lam", [(0, 0.01), (1, 0.1)])
def test_sparse_delta_forced(dims, ranks, mf, reg, lam):
    nnz = min(int(np.prod(dims)) // 3, 4000)
    phases(dims, ranks, nnz, 31, reg, lam, iters=2, mask_frac=mf, sparse=1)


# plan-specialised (NVRTC) core passes forced on/off across orders, plans and
# masks (prefix blocks for dense cores, live-fiber runs for sparse ones)
@pytest.mark.parametrize("dims,ranks,mf", [([20, 18, 16, 14], [8, 8, 8, 8], 0.9), ([9, 8, 8, 7, 7], [5, 5, 5, 5, 5], 0.0),
                                           ([30, 25], [4, 3], 0.2), ([7, 6, 5, 4, 3], [2, 2, 3, 2, 2], 0.2),
                                           ([40, 30, 20], [3, 5, 4], 0.3)])
@pytest.mark.parametrize("gen", [0, 1])
def test_core_gen_passes(dims, ranks, mf, gen):
    nnz = min(int(np.prod(dims)) // 3, 4000)
    phases(dims, ranks, nnz, 41, 0, 0.01, iters=2, mask_frac=mf, core_gen=gen)
    phases(dims, ranks, nnz, 42, 1, 0.1, iters=1, mask_frac=mf, core_gen=gen)


def test_sparse_delta_heavy_rows():
    phases([3, 60, 60], [5, 5, 5], 9000, 18, 0, 0.01, iters=1, sparse=1)
    # heavy rows in the LAST mode: their residual after k_heavy's solve
    # (k_rowpass_delta<kResid>) feeds the core sweep
    phases([60, 60, 3], [5, 5, 5], 9000, 19, 0, 0.01, iters=2, sparse=1)
    phases([40, 30, 25, 3], [3, 2, 4, 2], 9000, 21, 1, 0.05, iters=1, sparse=1, mask_frac=0.2)
    phases([12, 40, 30], [5, 5, 5], 8000, 20, 1, 0.05, iters=1, skew=1.6, sparse=1)


def test_config5_ranks():
    phases([9, 8, 8, 7, 7], [5, 5, 5, 5, 5], 4000, 15, 0, 0.01, iters=1)


@pytest.mark.parametrize("dims,ranks", [([30, 25], [4, 3]), ([6, 5, 4, 3], [2, 3, 2, 2]),
                                        ([7, 6, 5, 4, 3], [2, 2, 3, 2, 2]), ([5, 4, 3], [2, 3, 2])])
def test_generic_shapes(dims, ranks):
    nnz = min(int(np.prod(dims)) // 3, 800)
    phases(dims, ranks, nnz, 16, 0, 0.05, mask_frac=0.2)
    phases(dims, ranks, nnz, 17, 1, 0.2, mask_frac=0.2)


@pytest.mark.parametrize("ranks", [[5, 5, 5], [3, 2, 2]])
def test_heavy_rows_split_across_chunks(ranks):
    # mode-0 rows hold ~3000-5000 entries: several kChunk work items per row
    phases([3, 60, 60], ranks, 9000, 18, 0, 0.01, iters=1)
    phases([3, 60, 60], ranks, 9000, 19, 1, 0.05, iters=1)


@pytest.mark.parametrize("dims,ranks", [([400, 30, 20], [5, 5, 5]), ([300, 40, 30], [10, 10, 5]),
                                        ([200, 20, 18, 16], [8, 8, 8, 8])])
def test_short_rows_lane_per_row(dims, ranks):
    # mode-0 rows hold ~1-40 entries: the lane-per-row statistics kernel
    # (k_rowpass_tiny) for rows <= 32 entries, the chunk kernel for the rest
    phases(dims, ranks, 5000, 51, 0, 0.01, iters=2, mask_frac=0.1)
    phases(dims, ranks, 5000, 52, 1, 0.05, iters=1, mask_frac=0.1)


def test_skewed_rows():
    phases([12, 40, 30], [5, 5, 5], 8000, 20, 0, 0.01, iters=1, skew=1.6)


def test_empty_rows_policies():
    # rows 2 and 4 of mode 0 have no entries
    dims, ranks = [6, 5, 4], [2, 2, 2]
    rng = np.random.default_rng(3)
    cells = [c for c in range(120) if (c // 20) not in (2, 4)]
    cells = np.sort(rng.choice(cells, 40, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    values = rng.uniform(-1, 2, 40)
    m = st.init_random(dims, ranks, 8)
    m.factors[0][2, 1] = 0.0
    m.factor_masks[0][2, 1] = 1
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    dev.update_all_factors(0, 0.1)
    got = dev.get_model()
    assert np.array_equal(got.factors[0][2], m.factors[0][2])  # LF: untouched
    assert np.array_equal(got.factors[0][4], m.factors[0][4])
    dev.set_model(m)
    dev.update_all_factors(1, 0.1)
    got = dev.get_model()
    assert got.factors[0][2, 0] == 0.0 and got.factors[0][2, 1] == 0.0  # L1: zeroed / masked
    assert np.all(got.factors[0][4] == 0.0)


def test_known_answers_one_cell():
    # tests/test_updates.cpp:186-220
    def one(xv):
        x = st.make_tensor([1, 1], [[0, 0]], [xv])
        m = st.TuckerModel([1, 1], [1, 1], np.ones(1), np.zeros(1, np.uint8), [np.ones((1, 1)), np.ones((1, 1))],
                           [np.zeros((1, 1), np.uint8)] * 2)
        return x, m
    x, m = one(2.0)
    st.update_factor_row_lf(m, x, None, 0, 0, 1.0)
    assert abs(m.factors[0][0, 0] - 1.0) <= 1e-15
    x, m = one(2.0)
    st.update_factor_row_l1(m, x, None, 0, 0, 1.0)
    assert abs(m.factors[0][0, 0] - 1.5) <= 1e-15
    x, m = one(3.0)
    st.update_core_l1(m, x, 1.0)
    assert abs(m.core[0] - 2.5) <= 1e-15
    x, m = one(3.0)
    st.update_core_lf(m, x, 1.0)
    assert abs(m.core[0] - 1.5) <= 1e-15


def test_zero_denominator_policies():
    # tests/test_updates.cpp:239-272
    x = st.make_tensor([2, 2], [[0, 0], [1, 1]], [1.0, 2.0])
    base = st.init_random([2, 2], [2, 2], 9)
    base.core[2] = 0.0
    base.core[3] = 0.0
    m = base.copy()
    orig = m.factors[0][0, 1]
    st.update_factor_row_lf(m, x, None, 0, 0, 0.0)
    assert m.factors[0][0, 1] == orig
    m = base.copy()
    st.update_factor_row_lf(m, x, None, 0, 0, 0.5)
    assert m.factors[0][0, 1] == 0.0
    m = base.copy()
    st.update_factor_row_l1(m, x, None, 0, 0, 0.0)
    assert m.factors[0][0, 1] == 0.0
    m = base.copy()
    m.factors[0][0, 1] = 0.0
    m.factors[0][1, 1] = 0.0
    m.core[2] = 0.7
    m2 = m.copy()
    st.update_core_lf(m, x, 0.0)
    assert m.core[2] == 0.7
    st.update_core_l1(m2, x, 0.3)
    assert m2.core[2] == 0.7


def test_fully_pruned_fixed_point():
    x = st.make_tensor([2, 2], [[0, 0], [1, 1]], [1.0, 2.0])
    m = st.init_random([2, 2], [2, 2], 10)
    m.core[:] = 0
    m.core_mask[:] = 1
    for n in range(2):
        m.factors[n][:] = 0
        m.factor_masks[n][:] = 1
    before = m.copy()
    st.update_all_factors(m, x, None, 0, 0.1)
    st.update_core_lf(m, x, 0.1)
    st.update_all_factors(m, x, None, 1, 0.1)
    st.update_core_l1(m, x, 0.1)
    assert np.array_equal(m.core, before.core)
    for n in range(2):
        assert np.array_equal(m.factors[n], before.factors[n])


def test_perfect_fit_all_infinite():
    m = st.init_random([3, 3], [2, 2], 12)
    coords = np.array([[0, 0], [1, 2], [2, 1]], np.uint32)
    values = st.predict(m, coords)
    s = O.Session([3, 3], coords, values, [2, 2], "port")
    s.set_model(m.core, m.core_mask, m.factors, m.factor_masks)
    _, _, _, re_ref = s.compute_residuals(1)
    x = st.make_tensor([3, 3], coords, values)
    dev = st.Device(x, [2, 2])
    dev.set_model(m)
    res = dev.compute_residuals()
    if re_ref == 0.0 and res.re == 0.0:
        tab = dev.compute_responsibilities()
        assert np.all(np.isinf(tab.core))
        assert all(np.all(np.isinf(f)) for f in tab.factors)


def test_prune_ties_floor_saturation():
    # tests/test_pruning.cpp:179-231 on the device radix select
    m = st.init_random([2, 2], [2, 2], 3)
    t = st.ResponsibilityTable(np.array([0.5, 0.2, 0.2, 0.9]),
                               [np.array([0.1, 0.4, 0.4, 0.4]), np.array([0.7, 0.6, 0.5, 0.4])])
    c = st.prune_step(m, t, 0.5)
    assert (c.core, c.factors, c.total()) == (2, [2, 2], 6)
    assert list(m.core_mask) == [0, 1, 1, 0] and m.core[1] == 0.0 and m.core[2] == 0.0
    assert list(m.factor_masks[0].reshape(-1)) == [1, 1, 0, 0]
    assert list(m.factor_masks[1].reshape(-1)) == [0, 0, 1, 1]
    m = st.init_random([3, 1], [1, 1], 4)
    t = st.ResponsibilityTable(np.array([0.5]), [np.array([0.3, 0.2, 0.1]), np.array([0.4])])
    c = st.prune_step(m, t, 0.4)
    assert (c.core, c.factors) == (0, [1, 0])
    assert list(m.factor_masks[0].reshape(-1)) == [0, 0, 1]
    t.factors[0] = np.array([0.3, 0.2, np.inf])
    c = st.prune_step(m, t, 0.9)
    assert c.factors[0] == 2
    c = st.prune_step(m, t, 0.9)
    assert c.factors[0] == 0
    with pytest.raises(ValueError):
        st.prune_step(m, t, 1.0)
    with pytest.raises(ValueError):
        st.prune_step(m, t, -0.1)
    m2 = st.init_random([3, 1], [1, 1], 4)
    t2 = st.ResponsibilityTable(np.array([0.5]), [np.array([0.3, 0.2, 0.1]), np.array([0.4])])
    assert st.prune_step(m2, t2, 0.0).total() == 0
    assert st.masked_fraction(m2) == 0.0


def test_prune_negative_zero_and_many_ties():
    rng = np.random.default_rng(5)
    dims, ranks = [400, 3], [5, 1]
    m = st.init_random(dims, ranks, 1)
    resp = np.round(rng.random(2000) * 4) / 4  # heavy ties
    resp[::7] = -0.0
    resp[::11] = 0.0
    s = O.Session(dims, np.zeros((1, 2), np.uint32), np.ones(1), ranks, "port")
    s.set_model(m.core, m.core_mask, m.factors, m.factor_masks)
    tab = st.ResponsibilityTable(np.array([0.3]), [resp, np.array([0.1, 0.2, 0.3])])
    for pr in (0.1, 0.33, 0.5, 0.77):
        c = st.prune_step(m, tab, pr)
        rc = s.prune_step(pr, tab.core, tab.factors)
        assert [c.core] + c.factors == [int(v) for v in rc]
        _, cm, fs, ms = s.get_model()
        assert np.array_equal(m.factor_masks[0].reshape(-1), ms[0].reshape(-1))
        assert np.array_equal(m.factor_masks[1].reshape(-1), ms[1].reshape(-1))


def test_errors_match_reference():
    with pytest.raises(ValueError, match="duplicate"):
        st.Device(st.SparseTensor([3, 3], np.array([[0, 1], [0, 1]], np.uint32), np.ones(2)), [1, 1])
    with pytest.raises(ValueError, match="out of bounds"):
        st.Device(st.SparseTensor([3, 3], np.array([[0, 3]], np.uint32), np.ones(1)), [1, 1])
    x = st.make_tensor([2, 2], [[0, 1]], [0.0])
    m = st.init_random([2, 2], [1, 1], 1)
    with pytest.raises(ValueError, match="zero-norm"):
        st.compute_residuals(m, x)
    m3 = st.init_random([2, 3], [1, 1], 1)
    with pytest.raises(ValueError, match="shape mismatch"):
        st.update_all_factors(m3, x, None, 0, 0.1)


def test_masked_never_written_and_monotone():
    dims, ranks = [20, 15, 10], [3, 3, 3]
    coords, values, m = random_instance(dims, ranks, 600, 26, mask_frac=0.2)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    for reg, lam in ((0, 0.01), (1, 0.3)):
        dev.update_all_factors(reg, lam)
        dev.update_core(reg, lam)
    got = dev.get_model()
    assert np.array_equal(got.core_mask, m.core_mask)
    assert np.all(got.core[m.core_mask == 1] == 0.0)
    for n in range(3):
        assert np.all(got.factors[n][m.factor_masks[n] == 1] == 0.0)
    prev = [got.core_mask.copy()] + [k.copy() for k in got.factor_masks]
    for _ in range(4):
        dev.compute_residuals()
        dev.compute_responsibilities(want=False)
        dev.prune_step(0.1)
        now = dev.get_model()
        cur = [now.core_mask] + list(now.factor_masks)
        for a, b in zip(prev, cur):
            assert np.all(b >= a)
        prev = [c.copy() for c in cur]


def test_bit_identical_reruns():
    dims, ranks = [50, 40, 30], [5, 5, 5]
    coords, values, m = random_instance(dims, ranks, 4000, 27, mask_frac=0.1)
    x = st.make_tensor(dims, coords, values)
    outs = []
    for _ in range(2):
        dev = st.Device(x, ranks)
        dev.set_model(m)
        re = [dev.cd_iteration(0, 0.01) for _ in range(3)]
        dev.compute_responsibilities(want=False)
        dev.prune_step(0.2)
        re.append(dev.cd_iteration(0, 0.01))
        outs.append((re, dev.get_model()))
        dev.close()
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1].core, outs[1][1].core)
    for n in range(3):
        assert np.array_equal(outs[0][1].factors[n], outs[1][1].factors[n])


def test_evaluate_and_predict_vs_oracle():
    dims, ranks = [40, 30, 20], [5, 5, 5]
    coords, values, m = random_instance(dims, ranks, 2000, 28)
    s = O.Session(dims, coords, values, ranks, "port")
    s.set_model(m.core, m.core_mask, m.factors, m.factor_masks)
    _, _, _, re = s.compute_residuals(1)
    x = st.make_tensor(dims, coords, values)
    assert abs(st.evaluate_test(m, x) - re) <= 1e-6 * re
    assert_close(st.predict(m, coords), s.reconstruct(coords), "predict")


def test_cd_iteration_trajectory_vs_oracle():
    """Unsynced trajectory: 5 CD iterations (fit's loop body) stay within tolerance."""
    dims, ranks = [60, 50, 40], [5, 5, 5]
    coords, values, m = random_instance(dims, ranks, 5000, 29, lo=0.0, hi=1.0)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    s = oracle_session(dims, ranks, coords, values, m)
    for _ in range(5):
        re = dev.cd_iteration(0, 0.01)
        re_ref = s.cd_iteration(0, 0.01, 1)
        assert abs(re - re_ref) <= 1e-6 * re_ref
    got, want = dev.get_model(), model_of(s, dims, ranks)
    assert_close(got.core, want.core, "core after 5 iterations")
    for n in range(3):
        assert_close(got.factors[n], want.factors[n], f"factor{n} after 5 iterations")


@pytest.mark.parametrize("dims,ranks,mf,pr", [([24, 20, 18, 16], [8, 8, 8, 8], 0.9, 0.05),
                                              ([9, 8, 8, 7, 7], [5, 5, 5, 5, 5], 0.0, 0.2)])
def test_auto_kernel_switch_trajectory_vs_oracle(dims, ranks, mf, pr):
    """Auto mode on rank-specialised 4/5-mode shapes: sweep 1 runs the
    precompiled kernels, sweep 2 compiles the mask's NVRTC kernels (generated
    core passes; the mask-specialised delta for the 90 %-masked core), a prune
    changes the mask (precompiled again for one sweep, then recompiled) -- the
    whole trajectory stays on the oracle's."""
    coords, values, m = random_instance(dims, ranks, 5000, 61, mask_frac=mf, lo=0.0, hi=1.0)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    s = oracle_session(dims, ranks, coords, values, m)
    for t in range(6):
        re = dev.cd_iteration(0, 0.01)
        re_ref = s.cd_iteration(0, 0.01, 1)
        assert abs(re - re_ref) <= 1e-6 * re_ref, t
        if t == 2:
            before = model_of(s, dims, ranks)
            dev.compute_responsibilities(want=False)
            s.compute_residuals(1)
            rc, _ = s.compute_responsibilities(1)
            counts = dev.prune_step(pr)
            ref_counts = s.prune_step(pr)
            assert 0 < counts.core < int(np.sum(m.core_mask == 0))  # the core survives the prune
            assert [counts.core] + counts.factors == [int(c) for c in ref_counts]
            want = model_of(s, dims, ranks)
            assert_masks(dev.get_model().core_mask, want.core_mask, rc, before.core_mask, "core mask")
            # near-threshold ties may pick different cells (within tolerance):
            # continue both from the oracle's pruned model
            dev.set_model(want)
    got, want = dev.get_model(), model_of(s, dims, ranks)
    assert_close(got.core, want.core, "core")
    for n in range(len(dims)):
        assert_close(got.factors[n], want.factors[n], f"factor{n}")


@pytest.mark.parametrize("ranks", [[3, 3, 2], [5, 5, 5], [2, 3, 2, 2]])
def test_iteration_re_after_core_fully_pruned(ranks):
    """A prune that masks every core cell (k is floored against the block size,
    masked cells included): the next iteration's RE is that of the zero
    reconstruction, 1.0, exactly as the reference's."""
    dims = [20, 18, 16, 14][: len(ranks)]
    coords, values, m = random_instance(dims, ranks, 1500, 71, lo=0.0, hi=1.0)
    m.core_mask[:] = 1
    m.core_mask.reshape(-1)[0] = 0
    m.core[m.core_mask == 1] = 0.0
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    s = oracle_session(dims, ranks, coords, values, m)
    dev.cd_iteration(0, 0.01)
    s.cd_iteration(0, 0.01, 1)
    dev.compute_responsibilities(want=False)
    s.compute_residuals(1)
    s.compute_responsibilities(1)
    assert dev.prune_step(0.5).core == int(s.prune_step(0.5)[0]) == 1
    for _ in range(2):
        re, re_ref = dev.cd_iteration(0, 0.01), s.cd_iteration(0, 0.01, 1)
        assert re_ref == 1.0 and abs(re - re_ref) <= 1e-12, (re, re_ref)


@pytest.mark.parametrize("dims,ranks,mf", [([60, 50, 40], [5, 5, 5], 0.0), ([60, 50, 40], [10, 10, 5], 0.0),
                                           ([20, 18, 16, 14], [8, 8, 8, 8], 0.9),
                                           ([9, 8, 8, 7, 7], [5, 5, 5, 5, 5], 0.0)])
def test_iteration_graph_replay_bit_identical(dims, ranks, mf):
    """From the fifth iteration with an unchanged mask on, an iteration is
    captured once as a CUDA graph and replayed -- the 3-mode all-prefix sweep
    and the general sweep (4-mode masked core: mask-specialised delta + plan-
    specialised passes; 5-mode dense) -- and must reproduce the stream path
    bit for bit (the stream path is forced by profiling, which disables
    graphs); a prune in between drops back to the stream path."""
    from paper_1904_02603_b200 import _lib
    coords, values, m = random_instance(dims, ranks, 6000 if len(dims) == 3 else 4000, 81, lo=0.0, hi=1.0,
                                        mask_frac=0.0)
    if mf > 0:
        cm = (np.random.default_rng(5).random(m.core.shape) < mf).astype(np.uint8)
        m.core[cm == 1] = 0.0
        m.core_mask = cm
    x = st.make_tensor(dims, coords, values)
    out = []
    for profile in (0, 1):
        dev = st.Device(x, ranks)
        _lib.lib().vest_ctx_profile(dev.h, profile)
        dev.set_model(m)
        before = _lib.lib().vest_launch_count()
        res = [dev.cd_iteration(0, 0.01) for _ in range(8)]
        launches = _lib.lib().vest_launch_count() - before
        dev.compute_responsibilities(want=False)
        dev.prune_step(0.1)
        res += [dev.cd_iteration(1, 0.05) for _ in range(8)]
        out.append((res, dev.get_model(), launches))
        dev.close()
    (ra, ma, la), (rb, mb, lb) = out
    assert ra == rb
    assert la == lb  # replays are counted like the launches they contain
    assert np.array_equal(ma.core, mb.core)
    for n in range(len(dims)):
        assert np.array_equal(ma.factors[n], mb.factors[n])
