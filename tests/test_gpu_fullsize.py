"""Parity at BASELINE.json's full sizes (configs 1-5), through checks whose cost
does not grow with the tensor (the CPU oracle cannot sweep
10^8 entries in test time):

* config 1 (CPU-runnable, 100k entries) runs BASELINE's whole protocol -- 10
  CD iterations then a prune at rate 0.5 -- against the oracle end to end;
* configs 2-5, per factor mode: rows are independent within a mode
  (updates.hpp:153-175), so the device's full-mode update of sampled rows
  (heavy multi-chunk rows, random rows, empty rows) must equal the oracle's
  update_factor_row on a session holding only those rows' entries and the
  same pre-update model;
* the core sweep: after an exact Gauss-Seidel sweep the LAST unmasked cell is
  stationary against the final residual (updates.hpp:211-236), checked in
  numpy over every observed entry;
* RE: the sweep's RE against an independent full reconstruction (predict);
* prune: the device's masks and counts after prune_step equal the oracle's
  prune_step applied to the same responsibility table and model
  (pruning.hpp:206-247).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_02603_b200 import _lib
from paper_1904_02603_b200 import sparsetuck as st
from parity import assert_close

pytestmark = pytest.mark.gpu

# BASELINE.json configs (bench.py CONFIGS carries the same numbers)
CONFIGS = {
    1: dict(dims=[1000] * 3, nnz=100_000, ranks=[5, 5, 5], lam=0.01, zipf=None, kind=0),
    2: dict(dims=[100_000] * 3, nnz=10_000_000, ranks=[10, 10, 10], lam=0.01, zipf=None, kind=0),
    3: dict(dims=[1_000_000, 200_000, 1000], nnz=50_000_000, ranks=[10, 10, 5], lam=0.1, zipf=[1.1, 1.1, 0.0],
            kind=1),
    4: dict(dims=[1_000_000] * 4, nnz=200_000_000, ranks=[8, 8, 8, 8], lam=0.01, zipf=None, kind=2,
            core_keep=0.1),
    5: dict(dims=[100_000] * 5, nnz=100_000_000, ranks=[5] * 5, lam=0.01, zipf=[1.0] * 5, kind=0),
}


def synth(c, seed):
    L = _lib.lib()
    dims = c["dims"]
    d = np.asarray(dims, np.uint64)
    z = np.asarray(c["zipf"] or [0.0] * len(dims), np.float64)
    coords = np.empty(c["nnz"] * len(dims), np.uint32)
    vals = np.empty(c["nnz"], np.float64)
    _lib.check(L.vest_synth(len(dims), _lib.ptr(d, _lib.u64p), c["nnz"], _lib.ptr(z, _lib.f64p), c["kind"], seed,
                            _lib.ptr(coords, _lib.u32p), _lib.ptr(vals, _lib.f64p)))
    return coords.reshape(c["nnz"], len(dims)), vals


def initial_model(c):
    m = st.init_random(c["dims"], c["ranks"], 7)
    if c.get("core_keep", 1.0) < 1.0:  # seeded core mask
        mask = (np.random.default_rng(44).random(m.core.shape) >= c["core_keep"]).astype(np.uint8)
        m.core[mask == 1] = 0.0
        m.core_mask = mask
    return m


def sample_rows(counts, rng, max_entries=400_000):
    """The heaviest row the oracle can update quickly (multi-chunk when the
    mode is skewed), four random rows and an empty row when there is one."""
    order = np.argsort(-counts, kind="stable")
    heavy = [int(r) for r in order if counts[r] <= max_entries][:1]
    rnd = [int(r) for r in rng.choice(len(counts), 4, replace=False)]
    empty = [int(r) for r in np.nonzero(counts == 0)[0][:1]]
    return sorted(set(heavy + rnd + empty))


def row_oracle(c, coords, vals, before, mode, rows, lam):
    sel = np.isin(coords[:, mode], np.asarray(rows, np.uint32))
    ses = O.Session(c["dims"], coords[sel], vals[sel], c["ranks"], "port")
    ses.set_model(before.core, before.core_mask, before.factors, before.factor_masks)
    for i in rows:
        ses.update_factor_row(0, mode, i, lam)
    return ses.get_model()[2][mode][rows]


def cell_products(m, coords, beta):
    p = np.ones(len(coords))
    for k, b in enumerate(beta):
        p *= m.factors[k][coords[:, k], b]
    return p


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_fullsize_sampled_rows_core_stationarity_prune(cfg):
    c = CONFIGS[cfg]
    coords, vals = synth(c, 1000 + cfg)
    x = st.SparseTensor(c["dims"], coords, vals)
    dev = st.Device(x, c["ranks"], 0)
    dev.set_model(initial_model(c))
    rng = np.random.default_rng(cfg)
    lam = c["lam"]
    # factor modes: sampled rows against the oracle
    for n in range(len(c["dims"])):
        before = dev.get_model()
        dev.update_factor_mode(n, 0, lam)
        after = dev.get_model()
        counts = np.bincount(coords[:, n], minlength=c["dims"][n])
        rows = sample_rows(counts, rng)
        ref = row_oracle(c, coords, vals, before, n, rows, lam)
        assert_close(after.factors[n][rows], ref, f"config {cfg} mode {n} rows {rows}")
        # rows outside the sample moved too (the mode was updated as a whole)
        assert not np.array_equal(after.factors[n], before.factors[n])
    # core sweep: the last unmasked cell is stationary against the final residual
    dev.update_core(0, lam)
    m = dev.get_model()
    live = np.nonzero(m.core_mask.reshape(-1) == 0)[0]
    last = int(live[-1])
    beta = np.unravel_index(last, c["ranks"])
    r = vals - dev.predict(coords)
    p = cell_products(m, coords, beta)
    g = float(m.core.reshape(-1)[last])
    num = float(np.dot(r + g * p, p))
    den = float(np.dot(p, p))
    g_star = num / (den + lam)
    assert abs(g - g_star) <= 1e-6 * max(abs(g_star), 1e-3 * np.abs(m.core).max()), (g, g_star)
    # RE of the sweep vs an independent reconstruction
    res = dev.compute_residuals()
    re_np = float(np.sqrt(np.dot(r, r)) / np.sqrt(np.dot(vals, vals)))
    assert abs(res.re - re_np) <= 1e-6 * re_np, (res.re, re_np)
    # prune: device selection vs the oracle's on the same table and model
    table = dev.compute_responsibilities()
    pre = dev.get_model()
    counts = dev.prune_step(0.3, table)
    post = dev.get_model()
    one = O.Session(c["dims"], coords[:1], vals[:1], c["ranks"], "port")
    one.set_model(pre.core, pre.core_mask, pre.factors, pre.factor_masks)
    rc = one.prune_step(0.3, table.core, table.factors)
    core_o, cm_o, fs_o, ms_o = one.get_model()
    assert [counts.core] + counts.factors == [int(v) for v in rc]
    assert np.array_equal(post.core_mask.reshape(-1), cm_o.reshape(-1))
    assert np.array_equal(post.core.reshape(-1), core_o.reshape(-1))
    for n in range(len(c["dims"])):
        assert np.array_equal(post.factor_masks[n].reshape(-1), ms_o[n].reshape(-1)), f"mode {n} masks"
        assert np.array_equal(post.factors[n].reshape(-1), fs_o[n].reshape(-1)), f"mode {n} values"
    dev.close()


def test_fullsize_config1_protocol_vs_oracle():
    """BASELINE config 1 end to end: 10 CD iterations, then prune at 0.5."""
    c = CONFIGS[1]
    coords, vals = synth(c, 1001)
    x = st.SparseTensor(c["dims"], coords, vals)
    dev = st.Device(x, c["ranks"], 0)
    m0 = initial_model(c)
    dev.set_model(m0)
    ses = O.Session(c["dims"], coords, vals, c["ranks"], "port")
    ses.set_model(m0.core, m0.core_mask, m0.factors, m0.factor_masks)
    for t in range(10):
        re = dev.cd_iteration(0, c["lam"])
        re_o = ses.cd_iteration(0, c["lam"], 8)
        assert abs(re - re_o) <= 1e-6 * re_o, (t, re, re_o)
    m = dev.get_model()
    core, cm, fs, ms = ses.get_model()
    assert_close(m.core, core, "core")
    for n in range(3):
        assert_close(m.factors[n], fs[n], f"factor {n}")
    table = dev.compute_responsibilities()
    ref_core, ref_f = ses.compute_responsibilities(8)
    counts = dev.prune_step(0.5, table)
    rc = ses.prune_step(0.5, ref_core, ref_f)
    assert [counts.core] + counts.factors == [int(v) for v in rc]
    dev.close()
