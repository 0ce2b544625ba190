"""vest_cd_iteration_host (the e2e entry point: host model in/out, factors read
back behind the later modes) is the same computation as set_model +
cd_iteration + get_model -- bit for bit -- including padded device rows
(odd ranks: ld = J + 1) and L1; and both agree with the oracle."""
import numpy as np
import pytest

from parity import assert_close

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")


def _instance(dims, nnz, seed):
    rng = np.random.default_rng(seed)
    cells = np.sort(rng.choice(int(np.prod(dims)), size=nnz, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    return st.make_tensor(dims, coords, rng.uniform(0.0, 1.0, len(cells)))


def _copy(m):
    return st.TuckerModel(list(m.dims), list(m.ranks), m.core.copy(), m.core_mask.copy(),
                          [f.copy() for f in m.factors], [k.copy() for k in m.factor_masks])


@pytest.mark.parametrize("ranks,reg", [([10, 10, 10], 0), ([5, 5, 5], 1), ([3, 5, 7], 0), ([4, 3, 2, 5], 0)])
def test_host_iteration_bitwise(ranks, reg, oracle_lib):
    dims = [40, 36, 30, 12][: len(ranks)]
    x = _instance(dims, 6000, 11)
    a = st.Device(x, ranks)
    b = st.Device(x, ranks)
    a.init_random(5)
    b.init_random(5)
    m_b = b.get_model()
    for it in range(3):
        m_a_in = a.get_model()
        a.set_model(m_a_in)
        re_a = a.cd_iteration(reg, 0.02)
        m_a = a.get_model()
        re_b = b.cd_iteration_host(m_b, reg, 0.02)
        assert re_a == re_b, (it, re_a, re_b)
        assert np.array_equal(m_a.core, m_b.core)
        for n in range(len(ranks)):
            assert np.array_equal(m_a.factors[n], m_b.factors[n]), (it, n)
    # and the host model matches the oracle's iteration from the same start
    from oracle import oracle as O
    s = O.Session(x.dims, x.coords, x.values, ranks, "port")
    s.init_random(5)
    for _ in range(3):
        s.cd_iteration(reg, 0.02)
    core, _, fs, _ = s.get_model()
    assert_close(m_b.core, core, "core", tol=1e-6)
    for n in range(len(ranks)):
        assert_close(m_b.factors[n], fs[n], f"factor{n}", tol=1e-6)


def test_host_iteration_rejects_bad_arrays():
    x = _instance([20, 20, 20], 800, 3)
    d = st.Device(x, [3, 3, 3])
    d.init_random(1)
    m = d.get_model()
    m.factors[0] = np.asfortranarray(m.factors[0])
    with pytest.raises(ValueError):
        d.cd_iteration_host(m, 0, 0.1)
