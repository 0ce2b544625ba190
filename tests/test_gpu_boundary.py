"""Drop-in boundary pieces beyond the CD sweep itself:
compute_row_stats / RowUpdateScratch (updates.hpp:17-30,64-79), the scratch
overloads of update_factor_row_{lf,l1} (:88,:113), partial_reconstruct
(tucker_model.hpp:136-154), and the tensor-context cache (rebuilt when the
tensor's contents change in place).  Checked against the C restatement
(bit-identical for the reference-order kernels)."""
import numpy as np
import pytest

from parity import assert_close
from test_gpu_oracle import oracle_session, random_instance

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")


CASES = [([30, 20, 10], [4, 3, 5], 900, 0.0), ([12, 9, 8, 7], [3, 4, 2, 3], 700, 0.3),
         ([9, 8, 7, 6, 5], [2, 3, 2, 2, 3], 600, 0.25), ([300, 4, 3], [5, 4, 3], 1000, 0.2)]


@pytest.mark.parametrize("dims,ranks,nnz,mask", CASES)
def test_row_stats_bit_identical(dims, ranks, nnz, mask):
    coords, values, m = random_instance(dims, ranks, nnz, 41, mask_frac=mask)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    ref = oracle_session(dims, ranks, coords, values, m)
    counts = [np.bincount(coords[:, n], minlength=dims[n]) for n in range(len(dims))]
    for n in range(len(dims)):
        rows = set(range(min(dims[n], 5)))
        rows |= {int(np.argmax(counts[n]))}  # the heaviest row
        empty = np.flatnonzero(counts[n] == 0)
        if len(empty):
            rows.add(int(empty[0]))
        for i in sorted(rows):
            got = dev.row_stats(n, i)
            want = ref.row_stats(n, i)
            for a, b in zip(got, want):
                assert np.array_equal(a, b), (n, i)
    dev.close()


@pytest.mark.parametrize("dims,ranks,nnz,mask", CASES)
def test_partial_reconstruct_bit_identical(dims, ranks, nnz, mask):
    coords, values, m = random_instance(dims, ranks, nnz, 43, mask_frac=mask)
    ref = oracle_session(dims, ranks, coords, values, m)
    q = coords[:50]
    total = np.zeros(len(q))
    for n in range(len(dims)):
        for j in range(ranks[n]):
            got = np.array([st.partial_reconstruct(m, a, n, j) for a in q[:3]])
            assert np.array_equal(got, ref.partial_reconstruct(q[:3], n, j))
            dev = st._model_device(m)
            batch = dev.partial_reconstruct(q, n, j)
            assert np.array_equal(batch, ref.partial_reconstruct(q, n, j))
            if n == 0:
                total += batch
    # summing the slices over j recovers the full reconstruction (tucker_model.hpp:133-135)
    full = ref.reconstruct(q)
    assert np.allclose(total, full, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        st._model_device(m).partial_reconstruct(q, 0, ranks[0])


@pytest.mark.parametrize("reg", [0, 1])
def test_scratch_overloads(reg):
    dims, ranks = [40, 6, 5], [4, 3, 3]
    coords, values, m = random_instance(dims, ranks, 400, 47, mask_frac=0.2)
    keep = coords[:, 0] != 7  # row 7 of mode 0 has no entries
    coords, values = coords[keep], values[keep]
    x = st.make_tensor(dims, coords, values)
    idx = st.build_mode_index(x)
    ref = oracle_session(dims, ranks, coords, values, m)
    counts = np.bincount(coords[:, 0], minlength=dims[0])
    empty = int(np.flatnonzero(counts == 0)[0])
    busy = int(np.argmax(counts))
    fn = st.update_factor_row_lf if reg == 0 else st.update_factor_row_l1
    for i in [busy, empty]:
        s = st.RowUpdateScratch()
        s.reset(ranks[0])
        s.gram[:] = 7.0  # sentinel: an LF update of an empty row must not touch the scratch
        want = ref.row_stats(0, i)
        fn(m, x, idx, 0, i, 0.05, s)
        ref.update_factor_row(reg, 0, i, 0.05)
        _, _, fs, _ = ref.get_model()
        assert_close(m.factors[0][i], fs[0][i], f"row {i}")  # the solve's arithmetic order differs
        if reg == 0 and i == empty:
            assert np.all(s.gram == 7.0)
        else:
            assert np.array_equal(s.delta, want[0])
            assert np.array_equal(s.gram.reshape(ranks[0], ranks[0]), want[1])
            assert np.array_equal(s.xdelta, want[2])
    # the rest of the model is untouched by a row update
    for n in (1, 2):
        assert np.array_equal(m.factors[n], ref.get_model()[2][n])
    others = np.setdiff1d(np.arange(dims[0]), [busy, empty])
    assert np.array_equal(m.factors[0][others], ref.get_model()[2][0][others])


def test_context_cache_follows_in_place_edits():
    """The tensor's cached device context (CSF + values in HBM) is rebuilt
    when coords/values are edited in place (no stale CSF)."""
    dims, ranks = [50, 40, 30], [3, 3, 3]
    coords, values, m = random_instance(dims, ranks, 1500, 53)
    x = st.make_tensor(dims, coords, values)
    re1 = st.reconstruction_error(m, x)
    x.values *= 2.0  # same buffer, new contents
    re2 = st.reconstruction_error(m, x)
    ref = oracle_session(dims, ranks, coords, x.values, m)
    want = ref.compute_residuals(1, want_r=False)[3]
    assert abs(re2 - want) <= 1e-12 * want and re2 != re1
    x.coords[:, 2] = (x.coords[:, 2] + 1) % dims[2]  # coordinates too (still distinct)
    re3 = st.reconstruction_error(m, x)
    ref = oracle_session(dims, ranks, x.coords, x.values, m)
    want = ref.compute_residuals(1, want_r=False)[3]
    assert abs(re3 - want) <= 1e-12 * want


def test_get_factor_rows():
    dims, ranks = [70, 9, 8], [5, 3, 4]
    coords, values, m = random_instance(dims, ranks, 300, 59)
    x = st.make_tensor(dims, coords, values)
    dev = st.Device(x, ranks)
    dev.set_model(m)
    dev.update_all_factors(0, 0.01)
    full = dev.get_model()
    for n in range(3):
        assert np.array_equal(dev.get_factor_rows(n, 2, 5), full.factors[n][2:7])
    with pytest.raises(ValueError):
        dev.get_factor_rows(0, 68, 5)
    dev.close()
