"""Pin the C restatement (oracle/vest_oracle.c) against the reference's own
outputs (tests/golden/*.npz, made by oracle/_ref from the unmodified reference
headers).  Integer/byte results must be identical; because the port keeps the
reference's loop and reduction orders, floating-point results are required to
be BIT-identical as well.  CPU only."""
import numpy as np
import pytest

from conftest import SEQ_CASES, golden


def _session(O, g, kind="port"):
    dims = [int(d) for d in g["dims"]]
    s = O.Session(dims, g["coords"], g["values"], [int(r) for r in g["ranks"]], kind)
    core = g["init_core"]
    fs = [g[f"init_factor{n}"] for n in range(len(dims))]
    ms = [g[f"init_fmask{n}"] for n in range(len(dims))]
    s.set_model(core, g["init_core_mask"], fs, ms)
    return s


def test_init_random_matches_reference(oracle_lib):
    g = golden("init_random")
    for k in range(int(g["ncases"])):
        dims = [int(d) for d in g[f"case{k}_dims"]]
        ranks = [int(r) for r in g[f"case{k}_ranks"]]
        s = oracle_lib.Session(dims, np.zeros((1, len(dims)), np.uint32), np.ones(1), ranks, "port")
        s.init_random(int(g[f"case{k}_seed"]))
        core, cm, fs, ms = s.get_model()
        assert np.array_equal(core, g[f"case{k}_core"])
        assert not cm.any()
        for n in range(len(dims)):
            assert np.array_equal(fs[n], g[f"case{k}_factor{n}"])
            assert not ms[n].any()


@pytest.mark.parametrize("case", SEQ_CASES)
def test_sequence_bit_identical(oracle_lib, case):
    g = golden(case)
    N = len(g["dims"])
    s = _session(oracle_lib, g)
    for n in range(N):
        off, ids = s.get_index(n)
        assert np.array_equal(off, g[f"index_offsets{n}"])
        assert np.array_equal(ids, g[f"index_ids{n}"])
    reg, lam = int(g["reg"]), float(g["lam"])
    prune_at = set(int(t) for t in g["prune_at"])
    for t in range(1, int(g["iters"]) + 1):
        s.update_all_factors(reg, lam, 2)
        _, _, fs, _ = s.get_model()
        for n in range(N):
            assert np.array_equal(fs[n], g[f"t{t}_factors_factor{n}"]), (t, n)
        s.update_core(reg, lam, 2)
        core, _, _, _ = s.get_model()
        assert np.array_equal(core, g[f"t{t}_core"]), t
        r, ss, xn, re = s.compute_residuals(2)
        assert np.array_equal(r, g[f"t{t}_r"])
        assert (ss, xn, re) == (g[f"t{t}_sum_sq"], g[f"t{t}_x_norm"], g[f"t{t}_re"])
        assert s.sparsity() == g[f"t{t}_sparsity"]
        if t in prune_at:
            rc, rf = s.compute_responsibilities(3)
            assert np.array_equal(rc, g[f"t{t}_resp_core"])
            for n in range(N):
                assert np.array_equal(rf[n], g[f"t{t}_resp_factor{n}"])
            counts = s.prune_step(float(g["pr"]))
            assert np.array_equal(counts, g[f"t{t}_prune_counts"])
            core, cm, fs, ms = s.get_model()
            assert np.array_equal(cm, g[f"t{t}_pruned_core_mask"])
            for n in range(N):
                assert np.array_equal(ms[n], g[f"t{t}_pruned_fmask{n}"])
            assert s.masked_fraction() == g[f"t{t}_masked_fraction"]
    s.normalize_columns()
    core, _, fs, _ = s.get_model()
    assert np.array_equal(core, g["normalized_core"])
    for n in range(N):
        assert np.array_equal(fs[n], g[f"normalized_factor{n}"])
    probe = g["probe_coords"]
    assert np.array_equal(s.reconstruct(probe), g["probe_recon"])
    for n in range(N):
        d = np.stack([s.compute_delta(c, n) for c in probe])
        assert np.array_equal(d, g[f"probe_delta{n}"])


# ---- known-answer tests restated from the reference suite --------------------
# tests/test_updates.cpp:186-220: one observed value on a 1x1 tensor, every model
# element 1; closed-form argmins 1.0 (ridge factor), 1.5 (lasso factor),
# 2.5 (lasso core, x=3), 1.5 (ridge core, x=3).
def _one_cell(O, x):
    s = O.Session([1, 1], np.zeros((1, 2), np.uint32), np.array([x]), [1, 1], "port")
    s.set_model(np.ones(1), np.zeros(1, np.uint8), [np.ones((1, 1)), np.ones((1, 1))],
                [np.zeros((1, 1), np.uint8)] * 2)
    return s


def test_known_answers(oracle_lib):
    s = _one_cell(oracle_lib, 2.0)
    s.update_factor_row(0, 0, 0, 1.0)
    assert abs(s.get_model()[2][0][0, 0] - 1.0) <= 1e-15
    s = _one_cell(oracle_lib, 2.0)
    s.update_factor_row(1, 0, 0, 1.0)
    assert abs(s.get_model()[2][0][0, 0] - 1.5) <= 1e-15
    s = _one_cell(oracle_lib, 3.0)
    s.update_core(1, 1.0, 1)
    assert abs(s.get_model()[0][0] - 2.5) <= 1e-15
    s = _one_cell(oracle_lib, 3.0)
    s.update_core(0, 1.0, 1)
    assert abs(s.get_model()[0][0] - 1.5) <= 1e-15


def test_prune_ties_floor_saturation(oracle_lib):
    # tests/test_pruning.cpp:179-231
    O = oracle_lib
    s = O.Session([2, 2], np.zeros((1, 2), np.uint32), np.ones(1), [2, 2], "port")
    s.init_random(3)
    c = s.prune_step(0.5, np.array([0.5, 0.2, 0.2, 0.9]),
                     [np.array([0.1, 0.4, 0.4, 0.4]), np.array([0.7, 0.6, 0.5, 0.4])])
    assert list(c) == [2, 2, 2]
    core, cm, fs, ms = s.get_model()
    assert list(cm) == [0, 1, 1, 0] and core[1] == 0.0 and core[2] == 0.0
    assert list(ms[0].reshape(-1)) == [1, 1, 0, 0]
    assert list(ms[1].reshape(-1)) == [0, 0, 1, 1]
    s = O.Session([3, 1], np.zeros((1, 2), np.uint32), np.ones(1), [1, 1], "port")
    s.init_random(4)
    c = s.prune_step(0.4, np.array([0.5]), [np.array([0.3, 0.2, 0.1]), np.array([0.4])])
    assert list(c) == [0, 1, 0]
    c = s.prune_step(0.9, np.array([0.5]), [np.array([0.3, 0.2, np.inf]), np.array([0.4])])
    assert c[1] == 2
    c = s.prune_step(0.9, np.array([0.5]), [np.array([0.3, 0.2, np.inf]), np.array([0.4])])
    assert c[1] == 0
    with pytest.raises(ValueError):
        s.prune_step(1.0, np.array([0.5]), [np.array([0.3, 0.2, 0.1]), np.array([0.4])])
    with pytest.raises(ValueError):
        s.prune_step(-0.1, np.array([0.5]), [np.array([0.3, 0.2, 0.1]), np.array([0.4])])


def test_empty_row_policies(oracle_lib):
    # tests/test_updates.cpp:222-237: LF leaves rows without entries untouched,
    # L1 zeroes their unmasked elements.
    O = oracle_lib
    coords = np.array([[0, 0], [1, 1]], np.uint32)
    s = O.Session([3, 2], coords, np.array([1.0, -2.0]), [2, 2], "port")
    s.init_random(8)
    before = s.get_model()[2][0].copy()
    s.update_factor_row(0, 0, 2, 0.1)
    assert np.array_equal(s.get_model()[2][0], before)
    core, cm, fs, ms = s.get_model()
    fs[0][2, 1] = 0.0
    ms[0][2, 1] = 1
    s.set_model(core, cm, fs, ms)
    s.update_factor_row(1, 0, 2, 0.1)
    f0 = s.get_model()[2][0]
    assert f0[2, 0] == 0.0 and f0[2, 1] == 0.0


def test_errors(oracle_lib):
    O = oracle_lib
    with pytest.raises(ValueError, match="duplicate"):
        O.Session([3, 3], np.array([[0, 1], [0, 1]], np.uint32), np.ones(2), [1, 1], "port")
    with pytest.raises(ValueError, match="out of bounds"):
        O.Session([3, 3], np.array([[0, 3]], np.uint32), np.ones(1), [1, 1], "port")
    s = O.Session([2, 2], np.array([[0, 1]], np.uint32), np.zeros(1), [1, 1], "port")
    with pytest.raises(ValueError, match="zero-norm"):
        s.compute_residuals()


def _ref_available(O):
    return O.available("reference")


@pytest.mark.parametrize("case", ["seq_543_l1_masked", "seq_4mode_l1", "seq_5mode_lf", "seq_2mode_lf"])
def test_row_stats_and_partial_reconstruct_match_reference(oracle_lib, case):
    """compute_row_stats (updates.hpp:64-79) and partial_reconstruct
    (tucker_model.hpp:136-154) of the port vs the reference itself, bit for
    bit, on the golden instances (masked cores, empty rows included)."""
    if not _ref_available(oracle_lib):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    g = golden(case)
    N = len(g["dims"])
    p = _session(oracle_lib, g, "port")
    r = _session(oracle_lib, g, "reference")
    rng = np.random.default_rng(3)
    for n in range(N):
        rows = list(range(min(int(g["dims"][n]), 6))) + list(rng.integers(0, int(g["dims"][n]), 6))
        for i in rows:
            a = p.row_stats(n, int(i))
            b = r.row_stats(n, int(i))
            for u, v in zip(a, b):
                assert np.array_equal(u, v), (case, n, i)
    coords = g["coords"][:40]
    for n in range(N):
        for j in range(int(g["ranks"][n])):
            assert np.array_equal(p.partial_reconstruct(coords, n, j), r.partial_reconstruct(coords, n, j))


def test_update_factor_mode_composes_update_all_factors(oracle_lib):
    """vo_update_factor_mode over modes 0..N-1 == the reference's
    update_all_factors (updates.hpp:157-175), bit for bit."""
    if not _ref_available(oracle_lib):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    for case in ["seq_543_l1_masked", "seq_4mode_l1"]:
        g = golden(case)
        p = _session(oracle_lib, g, "port")
        r = _session(oracle_lib, g, "reference")
        reg, lam = int(g["reg"]), float(g["lam"])
        for n in range(len(g["dims"])):
            p.update_factor_mode(reg, n, lam, 3)
        r.update_all_factors(reg, lam, 2)
        for a, b in zip(p.get_model()[2], r.get_model()[2]):
            assert np.array_equal(a, b)
