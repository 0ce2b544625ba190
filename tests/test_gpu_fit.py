"""fit() (trainer.hpp:103-168) end to end on the GPU against the reference's
own fit traces (tests/golden/fit_trace.npz, made by oracle/_ref), and the
prune-rate auto-search sweep (BASELINE config 5 protocol) against the oracle."""
import numpy as np
import pytest

from conftest import golden
from parity import assert_close

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")
from oracle import oracle as O  # noqa: E402


@pytest.mark.parametrize("tag,mode,target", [("manual", st.StopMode.Manual, 0.4), ("auto", st.StopMode.Auto, 0.0)])
def test_fit_matches_reference_trace(tag, mode, target):
    g = golden("fit_trace")
    dims = [int(d) for d in g["dims"]]
    ranks = [int(r) for r in g["ranks"]]
    x = st.make_tensor(dims, g["coords"], g["values"])
    cfg = st.TrainConfig(ranks=ranks, lam=0.01, mode=mode, target_sparsity=target, elbow_threshold=0.05,
                         schedule=st.PruneSchedule(0.02, 0.1), max_iters=25, tol=1e-7, seed=5,
                         normalize_output=True)
    r = st.fit(x, cfg)
    ref_re = g[f"{tag}_re"]
    assert r.report.iters == len(ref_re)
    got = np.array([it.re for it in r.report.iterations])
    assert np.allclose(got, ref_re, rtol=1e-6, atol=0)
    assert [int(it.pruned) for it in r.report.iterations] == [int(v) for v in g[f"{tag}_pruned"]]
    assert np.array_equal(np.array([it.sparsity for it in r.report.iterations]), g[f"{tag}_sparsity"])
    assert abs(r.report.final_re - float(g[f"{tag}_final_re"])) <= 1e-6 * float(g[f"{tag}_final_re"])
    assert_close(r.model.core, g[f"{tag}_core"], f"{tag} core")
    for n in range(3):
        assert_close(r.model.factors[n], g[f"{tag}_factor{n}"], f"{tag} factor{n}")


def test_auto_search_rates_vs_oracle():
    rng = np.random.default_rng(9)
    dims, ranks = [30, 25, 20, 15, 12], [3, 3, 2, 2, 2]
    cells = np.sort(rng.choice(int(np.prod(dims)), 4000, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    x = st.make_tensor(dims, coords, rng.uniform(0, 1, len(cells)))
    train, test = st.split_train_test(x, 0.1, 42)
    assert (train.nnz(), test.nnz()) == (3600, 400)
    dev = st.Device(train, ranks)
    dev.init_random(1)
    for _ in range(3):
        dev.cd_iteration(0, 0.01)
    model = dev.get_model()
    rates = [round(0.1 * k, 1) for k in range(1, 10)]
    res = st.auto_search(train, test, model, rates)
    for rr in res:
        s = O.Session(dims, train.coords, train.values, ranks, "port")
        s.set_model(model.core, model.core_mask, model.factors, model.factor_masks)
        s.compute_residuals(1)
        s.compute_responsibilities(1)
        counts = s.prune_step(rr.rate)
        _, _, _, re_train = s.compute_residuals(1)
        core, cm, fs, ms = s.get_model()
        t = O.Session(dims, test.coords, test.values, ranks, "port")
        t.set_model(core, cm, fs, ms)
        _, _, _, re_test = t.compute_residuals(1)
        assert [rr.pruned.core] + rr.pruned.factors == [int(c) for c in counts]
        assert abs(rr.train_re - re_train) <= 1e-6 * re_train
        assert abs(rr.test_re - re_test) <= 1e-6 * re_test


def test_noiseless_planted_re_trace_vs_reference():
    """A near-exact fit (x = a planted model's reconstruction, start = the
    planted model perturbed by 3e-6): the per-iteration RE follows the
    reference's exact compute_residuals (trainer.hpp:127) down to RE < 1e-6,
    where the 3-mode sweep's quadratic-form sum of squares would cancel
     -- the device falls back to the exact residual sum there."""
    kind = "reference" if O.available("reference") else "port"
    rng = np.random.default_rng(12)
    dims, ranks = [60, 50, 40], [3, 3, 3]
    cells = np.sort(rng.choice(int(np.prod(dims)), 12000, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    planted = st.init_random(dims, ranks, 3)
    p = O.Session(dims, coords, np.ones(len(cells)), ranks, kind)
    p.set_model(planted.core, planted.core_mask, planted.factors, planted.factor_masks)
    values = p.reconstruct(coords)
    x = st.make_tensor(dims, coords, values)
    m0 = planted.copy()
    for f in m0.factors:
        f *= 1.0 + 3e-6 * rng.standard_normal(f.shape)
    dev = st.Device(x, ranks)
    dev.set_model(m0)
    ref = O.Session(dims, coords, values, ranks, kind)
    ref.set_model(m0.core, m0.core_mask, m0.factors, m0.factor_masks)
    trace = []
    for t in range(40):
        re = dev.cd_iteration(0, 0.0)
        re_o = ref.cd_iteration(0, 0.0, 4)
        assert abs(re - re_o) <= 1e-6 * re_o, (t, re, re_o)
        trace.append(re)
        if re < 3e-7:
            break
    assert trace[-1] < 1e-6, trace
    assert all(r > 0.0 for r in trace)  # never clamped to 0 (StopController.should_prune, pruning.hpp:50)
