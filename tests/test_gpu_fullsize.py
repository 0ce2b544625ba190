"""Parity at BASELINE.json's full sizes (configs 1-5), against the oracle
(oracle/vest_oracle.c, pinned bit-exact to the reference by tests/test_oracle.py)
wherever the oracle finishes in test time, and otherwise against torch fp64
restatements of the reference's formulas over every observed entry:

* config 1 (100k entries): BASELINE's whole protocol -- 10 CD iterations, then
  responsibilities and a prune at rate 0.5 -- against the oracle end to end:
  model, RE trace, both responsibility tables, masks and counts;
* config 2 (10M entries): one full CD iteration from the same initial model
  and a prune event -- the WHOLE model, RE, every responsibility and every
  mask against the oracle (its sequential core sweep included);
* config 3 (50M entries, Zipf head rows of millions of entries): every factor
  of a full update_all_factors and the factor responsibility tables against
  the oracle; the core sweep, RE and core responsibilities against torch;
  masks against the oracle's prune_step on those tables;
* configs 4 and 5 (200M / 100M entries) with the steady-state NVRTC kernels
  forced on (config 4: mask-specialised delta; both: plan-specialised core
  passes): factor modes, whole, against the oracle's update of that mode from
  the same model (rows are independent within a mode, updates.hpp:153-175);
  one core sweep checked cell by cell against the exact sequential
  Gauss-Seidel conditions of updates.hpp:185-245 (Gram matrix and right-hand
  side formed in torch fp64 over every entry); the RE against torch.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_02603_b200 import _lib
from paper_1904_02603_b200 import sparsetuck as st
from parity import assert_close, assert_close_fp32, assert_masks, assert_resp

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1

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
    if c.get("core_keep", 1.0) < 1.0:  # seeded core mask (bench.core_mask)
        mask = (np.random.default_rng(44).random(m.core.size) >= c["core_keep"]).astype(np.uint8)
        mask = mask.reshape(m.core.shape)
        m.core[mask == 1] = 0.0
        m.core_mask = mask
    return m


def oracle_of(c, coords, vals, m):
    s = O.Session(c["dims"], coords, vals, c["ranks"], "port")
    s.set_model(m.core, m.core_mask, m.factors, m.factor_masks)
    return s


def compare_model(m, s, what):
    core, cm, fs, ms = s.get_model()
    assert_close(m.core, core, f"{what} core")
    for n in range(len(fs)):
        assert_close(m.factors[n], fs[n], f"{what} factor {n}")


def compare_prune(dev, s, pr, what):
    """responsibilities (pruning.hpp:181-191) and prune_step (:234-247) of the
    device vs the oracle on the same model: tables, masks, counts."""
    pre = dev.get_model()
    table = dev.compute_responsibilities()
    re_o = s.compute_residuals(THREADS, want_r=False)[3]
    ref_core, ref_f = s.compute_responsibilities(THREADS)
    assert abs(table.base_re - re_o) <= 1e-6 * re_o
    assert_resp(table.core, ref_core, f"{what} core resp")
    for n in range(len(ref_f)):
        assert_resp(table.factors[n], ref_f[n], f"{what} factor {n} resp")
    counts = dev.prune_step(pr)
    rc = s.prune_step(pr)
    assert [counts.core] + counts.factors == [int(v) for v in rc], what
    post = dev.get_model()
    core, cm, fs, ms = s.get_model()
    assert_masks(post.core_mask, cm, ref_core, pre.core_mask, f"{what} core mask")
    for n in range(len(fs)):
        assert_masks(post.factor_masks[n], ms[n], ref_f[n], pre.factor_masks[n], f"{what} factor {n} mask")
    # pruned positions hold exactly 0 (tucker_model.hpp:15-20); nonzero counts agree
    assert np.all(post.core.reshape(-1)[post.core_mask.reshape(-1) == 1] == 0.0)
    nz_dev = np.count_nonzero(post.core) + sum(np.count_nonzero(f) for f in post.factors)
    nz_ref = np.count_nonzero(core) + sum(np.count_nonzero(f) for f in fs)
    assert nz_dev == nz_ref, what


# ----------------------------------------------------------------- config 1 --
def test_fullsize_config1_protocol_vs_oracle():
    """BASELINE config 1 end to end: 10 CD iterations, then responsibilities
    and a prune at 0.5."""
    c = CONFIGS[1]
    coords, vals = synth(c, 1001)
    x = st.SparseTensor(c["dims"], coords, vals)
    dev = st.Device(x, c["ranks"], 0)
    m0 = initial_model(c)
    dev.set_model(m0)
    ses = oracle_of(c, coords, vals, m0)
    for t in range(10):
        re = dev.cd_iteration(0, c["lam"])
        re_o = ses.cd_iteration(0, c["lam"], THREADS)
        assert abs(re - re_o) <= 1e-6 * re_o, (t, re, re_o)
    compare_model(dev.get_model(), ses, "config 1 after 10 iterations")
    compare_prune(dev, ses, 0.5, "config 1 prune 0.5")
    compare_model(dev.get_model(), ses, "config 1 after the prune")
    dev.close()


# ------------------------------------------------------------ configs 2, 3 --
def test_fullsize_config2_iteration_and_prune_whole_model():
    """Config 2: one full CD iteration (trainer.hpp:121-127) and a prune event
    on the full tensor -- the whole model, RE, both responsibility tables and
    every mask against the oracle (its sequential core sweep included)."""
    c = CONFIGS[2]
    coords, vals = synth(c, 1002)
    x = st.SparseTensor(c["dims"], coords, vals)
    dev = st.Device(x, c["ranks"], 0)
    m0 = initial_model(c)
    dev.set_model(m0)
    ses = oracle_of(c, coords, vals, m0)
    re = dev.cd_iteration(0, c["lam"])
    re_o = ses.cd_iteration(0, c["lam"], THREADS)
    assert abs(re - re_o) <= 1e-6 * re_o, (re, re_o)
    compare_model(dev.get_model(), ses, "config 2 iteration 1")
    compare_prune(dev, ses, 0.3, "config 2 prune 0.3")
    dev.close()


def test_fullsize_config3_zipf_heads_whole_model():
    """Config 3 (50M entries; Zipf(1.1) head rows of millions of entries --
    the split-row k_heavy path -- and a long tail of short rows -- the
    lane-per-row kernel): every factor of one full update_all_factors and the
    factor responsibility tables against the oracle; the core sweep against the
    exact sequential Gauss-Seidel conditions, the RE and the core
    responsibilities (pruning.hpp:98-134) against torch fp64 over every entry;
    the prune masks against the oracle's prune_step on those tables."""
    c = CONFIGS[3]
    coords, vals = synth(c, 1003)
    assert np.bincount(coords[:, 0]).max() > 1_000_000  # the head rows really are multi-chunk rows
    x = st.SparseTensor(c["dims"], coords, vals)
    dev = st.Device(x, c["ranks"], 0)
    m0 = initial_model(c)
    dev.set_model(m0)
    ses = oracle_of(c, coords, vals, m0)
    lam = c["lam"]
    dev.update_all_factors(0, lam)
    ses.update_all_factors(0, lam, THREADS)
    mid = dev.get_model()
    fs_o = ses.get_model()[2]
    for n in range(3):
        assert_close(mid.factors[n], fs_o[n], f"config 3 factor {n}")
    dev.set_model(model_from(ses, c))  # the sweep starts from the oracle's factors
    before = dev.get_model()
    dev.update_core(0, lam)
    after = dev.get_model()
    live = np.flatnonzero(before.core_mask.reshape(-1) == 0)
    t = torch_core_stats(c, coords, vals, after.factors, after.core, live, np.arange(len(live)), 2_000_000)
    check_gs(t, before.core, after.core, live, lam, "config 3")
    res = dev.compute_residuals()
    assert abs(res.re - t["re"]) <= 1e-6 * t["re"], (res.re, t["re"])
    # responsibilities: core vs torch's closed form of pruning.hpp:127-128, factors vs the oracle
    table = dev.compute_responsibilities()
    ref_core = core_resp_from(t, after.core, after.core_mask, live)
    assert_resp(table.core, ref_core, "config 3 core resp")
    ses.set_model(after.core, after.core_mask, after.factors, after.factor_masks)
    _, _, _, re_o = ses.compute_residuals(THREADS, want_r=False)
    assert abs(re_o - res.re) <= 1e-6 * re_o
    ref_f = ses.compute_responsibilities(THREADS)[1]
    for n in range(3):
        assert_resp(table.factors[n], ref_f[n], f"config 3 factor {n} resp")
    pre = dev.get_model()
    counts = dev.prune_step(0.3)
    rc = ses.prune_step(0.3, ref_core, ref_f)
    assert [counts.core] + counts.factors == [int(v) for v in rc]
    post = dev.get_model()
    _, cm_o, _, ms_o = ses.get_model()
    assert_masks(post.core_mask, cm_o, ref_core, pre.core_mask, "config 3 core mask")
    for n in range(3):
        assert_masks(post.factor_masks[n], ms_o[n], ref_f[n], pre.factor_masks[n], f"config 3 factor {n} mask")
    dev.close()


# ------------------------------------------------------- torch fp64 checks --
def torch_core_stats(c, coords, vals, factors, core, live, check_pos, chunk):
    """Over every observed entry, in torch fp64 (independent of the library's
    kernels): P = the unmasked cells' products, H = P^T P (rows check_pos),
    b = P^T x, and for g = core: r = x - P g, S = r.r, cr = P^T r,
    d = column sums of P^2, re = sqrt(S) / ||x||."""
    import torch

    dev = torch.device("cuda")
    N = len(c["dims"])
    betas = np.stack(np.unravel_index(live, c["ranks"]), 1)
    F = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in factors]
    B = [torch.from_numpy(betas[:, k].astype(np.int64)).to(dev) for k in range(N)]
    g = torch.from_numpy(core.reshape(-1)[live].copy()).to(dev)
    sel = torch.from_numpy(np.asarray(check_pos, np.int64)).to(dev)
    L = len(live)
    z = dict(dtype=torch.float64, device=dev)
    H = torch.zeros(len(check_pos), L, **z)
    b, cr, d = torch.zeros(L, **z), torch.zeros(L, **z), torch.zeros(L, **z)
    ss = torch.zeros((), **z)
    xx = torch.zeros((), **z)
    for lo in range(0, len(vals), chunk):
        cc = torch.from_numpy(coords[lo:lo + chunk].astype(np.int64)).to(dev)
        xv = torch.from_numpy(vals[lo:lo + chunk]).to(dev)
        P = torch.ones(len(xv), L, **z)
        for k in range(N):
            P *= F[k][cc[:, k]][:, B[k]]
        H += P[:, sel].T @ P
        b += P.T @ xv
        r = xv - P @ g
        cr += P.T @ r
        d += (P * P).sum(0)
        ss += r @ r
        xx += xv @ xv
        del P
    return {"H": H.cpu().numpy(), "b": b.cpu().numpy(), "cr": cr.cpu().numpy(), "d": d.cpu().numpy(),
            "S": float(ss), "re": float(torch.sqrt(ss) / torch.sqrt(xx)), "xnorm": float(torch.sqrt(xx)),
            "pos": np.asarray(check_pos)}


def check_gs(t, core_old, core_new, live, lam, what):
    """The reference's core sweep (updates.hpp:185-245) sets the unmasked cells
    q in row-major order to num_q / (den_q + lambda) against the residual that
    carries every earlier update.  With dg = g_new - g_old:
        num_q = b_q - (H g_new)_q + sum_{q' >= q} H[q, q'] dg_q' + g_old_q H[q, q]."""
    H, b = t["H"], t["b"]
    g_old = core_old.reshape(-1)[live]
    g_new = core_new.reshape(-1)[live]
    dg = g_new - g_old
    pos = t["pos"]
    exp = np.empty(len(pos))
    for i, q in enumerate(pos):
        num = b[q] - H[i] @ g_new + H[i, q:] @ dg[q:] + g_old[q] * H[i, q]
        exp[i] = num / (H[i, q] + lam)
    got = g_new[pos]
    floor = 1e-3 * np.abs(core_new).max()
    err = np.abs(got - exp) / np.maximum(np.abs(exp), floor)
    assert err.max() <= 1e-6, f"{what}: core cell {live[pos[int(np.argmax(err))]]} off by {err.max():.3e}"
    dead = np.setdiff1d(np.arange(core_new.size), live)
    assert np.all(core_new.reshape(-1)[dead] == 0.0)


def core_resp_from(t, core, core_mask, live):
    """compute_core_responsibilities (pruning.hpp:98-134):
    acc = sum_e (r_e + g p_e)^2 = S + 2 g cr + g^2 d; resp = (sqrt(acc)/||x|| - re)/re."""
    resp = np.full(core.size, np.inf)
    re = t["re"]
    if re == 0.0:
        return resp
    g = core.reshape(-1)[live]
    acc = t["S"] + g * (2.0 * t["cr"] + g * t["d"])
    resp[live] = (np.sqrt(np.maximum(acc, 0.0)) / t["xnorm"] - re) / re
    resp[core_mask.reshape(-1) == 1] = np.inf
    return resp


# ------------------------------------------------------------ configs 4, 5 --
@pytest.mark.parametrize("cfg", [4, 5])
def test_fullsize_steady_state_kernels(cfg):
    c = CONFIGS[cfg]
    coords, vals = synth(c, 1000 + cfg)
    x = st.SparseTensor(c["dims"], coords, vals)
    dev = st.Device(x, c["ranks"], 0)
    if cfg == 4:  # pruned core: the NVRTC mask-specialised delta (vest_sparse.cu) is its steady state
        dev.set_sparse_delta(1)
    dev.set_core_gen(1)  # the NVRTC plan-specialised core passes (vest_core_gen.cu)
    m0 = initial_model(c)
    dev.set_model(m0)
    lam = c["lam"]
    if cfg == 4:
        # every factor mode, whole, against the oracle's update of that mode
        ses = oracle_of(c, coords, vals, m0)
        for n in range(len(c["dims"])):
            dev.update_factor_mode(n, 0, lam)
            ses.update_factor_mode(0, n, lam, THREADS)
            assert_close(dev.get_model().factors[n], ses.get_model()[2][n], f"config 4 factor mode {n}")
            dev.set_model(model_from(ses, c))  # the next mode starts from identical factors
        del ses
    else:
        # config 5 (dense 3125-cell core): the oracle's delta costs ~8 us per
        # entry and a row is serial in it, so mode 0 is checked on rows whose
        # oracle update is tractable -- Zipf rows ranked 20..40 (hundreds of
        # thousands of entries each: many chunks, the k_heavy path), 300 random
        # rows and the empty rows -- on an oracle holding exactly their entries
        # (rows are independent within a mode, updates.hpp:153-175)
        counts = np.bincount(coords[:, 0], minlength=c["dims"][0])
        order = np.argsort(-counts, kind="stable")
        rng = np.random.default_rng(5)
        rows = np.unique(np.concatenate([order[20:40], rng.choice(c["dims"][0], 300, replace=False),
                                         np.flatnonzero(counts == 0)[:3]])).astype(np.int64)
        assert counts[rows].max() > 50_000
        sel = np.isin(coords[:, 0], rows.astype(np.uint32))
        ses = oracle_of(c, coords[sel], vals[sel], m0)
        dev.update_factor_mode(0, 0, lam)
        ses.update_factor_mode(0, 0, lam, THREADS)
        assert_close(dev.get_model().factors[0][rows], ses.get_model()[2][0][rows], "config 5 factor mode 0 rows")
        del ses
        for n in range(1, len(c["dims"])):
            dev.update_factor_mode(n, 0, lam)
    if cfg == 4:
        assert dev.sparse_delta_active()
    # one core sweep against the exact sequential Gauss-Seidel conditions
    before = dev.get_model()
    dev.update_core(0, lam)
    after = dev.get_model()
    live = np.flatnonzero(before.core_mask.reshape(-1) == 0)
    rng = np.random.default_rng(cfg)
    if len(live) <= 512:
        check_pos = np.arange(len(live))
    else:  # config 5: 3125 live cells; first, last and a random 250
        check_pos = np.unique(np.concatenate([[0, 1, len(live) - 1],
                                              rng.choice(len(live), 250, replace=False)]))
    t = torch_core_stats(c, coords, vals, after.factors, after.core, live, check_pos,
                         2_000_000 if cfg == 4 else 400_000)
    check_gs(t, before.core, after.core, live, lam, f"config {cfg}")
    res = dev.compute_residuals()
    assert abs(res.re - t["re"]) <= 1e-6 * t["re"], (res.re, t["re"])
    if cfg == 4:
        # the fp32 mode bench.py times for config 4 (fp32 factor gathers, fp32
        # chunk statistics, the mask-specialised delta contracted in fp32
        # arithmetic; statistics, solves and residuals fp64): the same sweep
        # within 1e-4 floored of the fp64 result, and a whole factor mode under
        # the fp32 criterion of SURVEY 8(c) (normwise 1e-4; tests/parity.py)
        dev.set_gather_f32(True)
        dev.set_model(before)
        dev.update_core(0, lam)
        f32 = dev.get_model()
        assert_close(f32.core, after.core, "config 4 core sweep, fp32 mode", tol=1e-4)
        dev.set_model(before)
        dev.update_factor_mode(1, 0, lam)
        f1_fp32 = dev.get_model().factors[1].copy()
        dev.set_gather_f32(False)
        dev.set_model(before)
        dev.update_factor_mode(1, 0, lam)
        fr, nw = assert_close_fp32(f1_fp32, dev.get_model().factors[1], "config 4 factor mode 1, fp32 mode")
        print(f"config 4 fp32 mode, factor mode 1 vs fp64: floored {fr:.3e} normwise {nw:.3e}")
    dev.close()


def model_from(ses, c):
    core, cm, fs, ms = ses.get_model()
    return st.TuckerModel(list(c["dims"]), list(c["ranks"]), core, cm, fs, ms)
