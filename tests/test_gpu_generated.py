"""The generated (NVRTC) factor-mode kernels: the fused contraction +
statistics + solve kernel (vest_sf_<n>) is bit-identical to the two-kernel
path it replaces (vest_sd_<n> writing delta to HBM, then k_rowpass_delta), and
the fp32-gather variant (BASELINE config 4 is the fp32 configuration) stays
within north_star's stated fp32 tolerance (1e-4) of the fp64 oracle."""
import numpy as np
import pytest

from parity import assert_close
from test_gpu_oracle import model_of, oracle_session, random_instance

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")

CASES = [([20, 18, 16, 14], [8, 8, 8, 8], 0.9, None), ([60, 50, 40], [5, 5, 5], 0.3, None),
         ([7, 6, 5, 4, 3], [2, 2, 3, 2, 2], 0.2, None), ([12, 40, 30], [5, 5, 5], 0.5, 1.6),
         ([30, 25], [4, 3], 0.2, None), ([40, 30, 20], [15, 3, 2], 0.5, None)]


@pytest.mark.parametrize("dims,ranks,mf,skew", CASES)
@pytest.mark.parametrize("reg,lam", [(0, 0.01), (1, 0.1)])
def test_fused_factor_update_bit_identical(dims, ranks, mf, skew, reg, lam):
    nnz = min(int(np.prod(dims)) // 3, 6000)
    coords, values, m = random_instance(dims, ranks, nnz, 61, mask_frac=mf, skew=skew)
    x = st.make_tensor(dims, coords, values)
    out = []
    for fused in (0, 1):
        dev = st.Device(x, ranks)
        dev.set_sparse_delta(1)
        dev.set_sparse_fused(fused)
        dev.set_model(m)
        for _ in range(2):
            dev.update_all_factors(reg, lam)
            dev.update_core(reg, lam)
        out.append(dev.get_model())
        dev.close()
    for n in range(len(dims)):
        assert np.array_equal(out[0].factors[n], out[1].factors[n]), n
    assert np.array_equal(out[0].core, out[1].core)
    s = oracle_session(dims, ranks, coords, values, m)
    for _ in range(2):
        s.update_all_factors(reg, lam, 1)
        s.update_core(reg, lam, 1)
    want = model_of(s, dims, ranks)
    for n in range(len(dims)):
        assert_close(out[1].factors[n], want.factors[n], f"factor {n}")


@pytest.mark.parametrize("dims,ranks,mf", [([30, 28, 26, 24], [8, 8, 8, 8], 0.9), ([20, 18, 16, 14, 12], [5] * 5, 0.0)])
def test_gather_f32_within_fp32_tolerance(dims, ranks, mf):
    """The fp32 mode (both generated kernel families): fp32-rounded factor
    operands, the mask-specialised delta contracted in fp32 arithmetic
    (VEST_SD_F32), fp64 statistics and solves -- model and RE within 1e-4 of
    the fp64 oracle after 3 iterations;
    the fp32 shadows follow every factor update (no stale copies)."""
    nnz = 8000
    coords, values, m = random_instance(dims, ranks, nnz, 67, mask_frac=mf)
    values = values.astype(np.float32).astype(np.float64)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_sparse_delta(1 if mf > 0 else -1)
    dev.set_core_gen(1)
    dev.set_gather_f32(True)
    dev.set_model(m)
    s = oracle_session(dims, ranks, coords, values, m)
    for t in range(3):
        re = dev.cd_iteration(0, 0.01)
        re_o = s.cd_iteration(0, 0.01, 1)
        assert abs(re - re_o) <= 1e-4 * re_o, (t, re, re_o)
    got, want = dev.get_model(), model_of(s, dims, ranks)
    assert_close(got.core, want.core, "core", tol=1e-4)
    for n in range(len(dims)):
        assert_close(got.factors[n], want.factors[n], f"factor {n}", tol=1e-4)
    # and it is a different computation from the fp64 path (the switch works)
    dev64 = st.Device(x, ranks)
    dev64.set_sparse_delta(1 if mf > 0 else -1)
    dev64.set_core_gen(1)
    dev64.set_model(m)
    for t in range(3):
        dev64.cd_iteration(0, 0.01)
    assert not np.array_equal(dev64.get_model().core, got.core)
    assert_close(dev64.get_model().core, want.core, "fp64 core")
