"""The data formats either side of the path against the
reference's own functions (oracle/_ref: the unmodified headers' load_coo /
save_coo / save_model / load_model through oracle/ref_shim.cpp): written files
byte-identical, parsed tensors/models identical, and errors with the same
exception class and message -- including files large enough to be parsed by
many threads, with the first error placed in a later chunk."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1904_02603_b200 import _lib
from paper_1904_02603_b200 import sparsetuck as st

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsparsetuck_ref.so")
u64p, u32p, f64p, u8p = (C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                         C.POINTER(C.c_uint8))


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    L = C.CDLL(REF_SO)
    L.vr_last_error.restype = C.c_char_p
    return L


def ref_load_coo(L, path, one_based=False):
    order, nnz = C.c_int(), C.c_uint64()
    rc = L.vr_load_coo(str(path).encode(), int(one_based), C.byref(order), C.byref(nnz), None, None, None)
    if rc:
        return rc, L.vr_last_error().decode()
    dims = np.zeros(order.value, np.uint64)
    coords = np.zeros(max(nnz.value * order.value, 1), np.uint32)
    values = np.zeros(max(nnz.value, 1))
    rc = L.vr_load_coo(str(path).encode(), int(one_based), C.byref(order), C.byref(nnz),
                       dims.ctypes.data_as(u64p), coords.ctypes.data_as(u32p), values.ctypes.data_as(f64p))
    n, k = nnz.value, order.value
    return 0, ([int(d) for d in dims], coords[: n * k].reshape(n, k), values[:n])


def ours_load_coo(path, one_based=False, threads=0):
    try:
        x = st.load_coo(path, one_based, threads)
    except ValueError as e:
        return 1, str(e)
    except _lib.VestError as e:
        return 2, str(e)
    return 0, (list(x.dims), x.coords, x.values)


def same_load(L, path, one_based=False, threads=0):
    a = ref_load_coo(L, path, one_based)
    b = ours_load_coo(path, one_based, threads)
    assert a[0] == b[0], (a, b)
    if a[0]:
        assert a[1] == b[1]
        return
    assert a[1][0] == b[1][0]
    assert np.array_equal(a[1][1], b[1][1])
    assert np.array_equal(a[1][2].view(np.uint64), b[1][2].view(np.uint64))  # bit-identical doubles


def awkward_values(rng, n):
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    v[::7] = 0.0
    v[1::11] = -0.0
    v[2::13] = np.round(v[2::13])
    v[3::17] = 5e-324  # subnormal
    v[4::19] = 1.0 / 3.0
    return v


def test_save_coo_byte_identical(ref, tmp_path):
    rng = np.random.default_rng(1)
    for order in (1, 3, 5):
        dims = [int(d) for d in rng.integers(1, 5000, order)]
        n = 20000
        cells = np.unique(np.stack([rng.integers(0, d, n) for d in dims], 1), axis=0)
        x = st.SparseTensor(dims, cells.astype(np.uint32), awkward_values(rng, len(cells)))
        a, b = tmp_path / f"ref{order}.coo", tmp_path / f"ours{order}.coo"
        d = np.asarray(dims, np.uint64)
        c = np.ascontiguousarray(x.coords).reshape(-1)
        assert ref.vr_save_coo(str(a).encode(), order, d.ctypes.data_as(u64p), x.nnz(), c.ctypes.data_as(u32p),
                               x.values.ctypes.data_as(f64p)) == 0
        st.save_coo(x, b)
        assert a.read_bytes() == b.read_bytes()
        same_load(ref, b)


def test_save_model_byte_identical(ref, tmp_path):
    rng = np.random.default_rng(2)
    dims, ranks = [300, 200, 150], [5, 4, 3]
    core = awkward_values(rng, int(np.prod(ranks)))
    factors = [awkward_values(rng, d * r).reshape(d, r) for d, r in zip(dims, ranks)]
    m = st.TuckerModel(dims, ranks, core, (core == 0).astype(np.uint8), factors,
                       [(f == 0).astype(np.uint8) for f in factors])
    ra, ob = tmp_path / "ref", tmp_path / "ours"
    d = np.asarray(dims, np.uint64)
    r = np.asarray(ranks, np.uint64)
    fp = (f64p * 3)(*[np.ascontiguousarray(f).ctypes.data_as(f64p) for f in factors])
    assert ref.vr_save_model(str(ra).encode(), 3, d.ctypes.data_as(u64p), r.ctypes.data_as(u64p),
                             core.ctypes.data_as(f64p), fp) == 0
    st.save_model(m, ob)
    names = sorted(os.listdir(ra))
    assert names == sorted(os.listdir(ob)) == ["core.coo", "factor_0.tsv", "factor_1.tsv", "factor_2.tsv"]
    for name in names:
        assert (ra / name).read_bytes() == (ob / name).read_bytes(), name
    # load_model: same model as the reference's, zeros become pruned
    back = st.load_model(ob)
    order = C.c_int()
    rd = np.zeros(3, np.uint64)
    rr = np.zeros(3, np.uint64)
    assert ref.vr_load_model(str(ra).encode(), C.byref(order), rd.ctypes.data_as(u64p), rr.ctypes.data_as(u64p),
                             None, None, None, None) == 0
    rcore = np.zeros(int(np.prod(ranks)))
    rcm = np.zeros(int(np.prod(ranks)), np.uint8)
    rf = [np.zeros((dd, rk)) for dd, rk in zip(dims, ranks)]
    rm = [np.zeros((dd, rk), np.uint8) for dd, rk in zip(dims, ranks)]
    assert ref.vr_load_model(str(ra).encode(), C.byref(order), rd.ctypes.data_as(u64p), rr.ctypes.data_as(u64p),
                             rcore.ctypes.data_as(f64p), rcm.ctypes.data_as(u8p),
                             (f64p * 3)(*[f.ctypes.data_as(f64p) for f in rf]),
                             (u8p * 3)(*[k.ctypes.data_as(u8p) for k in rm])) == 0
    assert back.dims == [int(v) for v in rd] and back.ranks == [int(v) for v in rr]
    assert np.array_equal(back.core.view(np.uint64), rcore.view(np.uint64))
    assert np.array_equal(back.core_mask, rcm)
    for n in range(3):
        assert np.array_equal(back.factors[n].view(np.uint64), rf[n].view(np.uint64))
        assert np.array_equal(back.factor_masks[n], rm[n])


CASES = {
    "plain": "0 1 2 0.5\n1 2 3 1.5\n",
    "comments_blank_crlf": "# a comment\n\n0 1 2 0.5\r\n  \t\n# dims: 4 5 6\n3 4 5 -2e-3\n",
    "two_dims_headers": "# dims: 4 5\n# dims: 6\n0 1 2 1\n",
    "dims_partial_token": "# dims: 4 5x 6\n0 1 1\n",
    "no_trailing_newline": "0 0 1\n1 1 2",
    "one_based": "1 1 1 1.0\n2 3 4 2.0\n",
    "stoll_prefix": "3x 1 0.5\n",
    "hex_value": "0 0 0x1.8p1\n",
    "header_only": "# dims: 3 4 5\n",
    "bad_coordinate": "0 1 2 0.5\n0 x 2 0.5\n",
    "negative": "0 1 2 0.5\n0 -1 2 0.5\n",
    "inconsistent": "0 1 2 0.5\n0 1 0.5\n",
    "bad_value": "0 1 2 0.5\n0 1 3 abc\n",
    "inf_value": "0 1 2 inf\n",
    "single_token": "5\n",
    "no_entries": "# just a comment\n\n",
    "dims_mismatch": "# dims: 3 4\n0 1 2 1\n",
    "out_of_bounds": "# dims: 2 2 2\n0 1 2 1\n",
    "duplicate": "0 1 2 1\n0 1 2 2\n",
    "overflow_coordinate": "99999999999999999999 1 1\n",
    "wrap_coordinate": "4294967297 1 1\n",
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_load_coo_cases(ref, tmp_path, case):
    p = tmp_path / f"{case}.coo"
    p.write_bytes(CASES[case].encode())
    same_load(ref, p, one_based=case == "one_based")
    if case == "one_based":
        same_load(ref, p, one_based=False)


def test_load_coo_many_threads(ref, tmp_path):
    """~6 MB of text -> many chunks; errors in a later chunk, a chunk starting
    with an inconsistent line, and comments between chunks."""
    rng = np.random.default_rng(3)
    n = 200000
    cells = np.unique(np.stack([rng.integers(0, 10 ** 6, n) for _ in range(3)], 1), axis=0)
    vals = awkward_values(rng, len(cells))
    lines = [f"{a} {b} {c} {v!r}" for (a, b, c), v in zip(cells.tolist(), vals.tolist())]
    for k in range(0, len(lines), 5000):
        lines.insert(k, "# dims: 1000000 1000000 1000000" if k == 0 else "# a comment")
    good = tmp_path / "good.coo"
    good.write_text("\n".join(lines) + "\n")
    for threads in (0, 1, 7):
        same_load(ref, good, threads=threads)
    for where, bad in [(len(lines) * 3 // 4, "1 2 x 0.5"), (len(lines) // 2, "1 2 0.5"),
                       (len(lines) - 2, "1 2 3 nan"), (len(lines) // 3, "7 7 -7 1")]:
        bl = list(lines)
        bl[where] = bad
        bl[min(where + 7, len(bl) - 1)] = "1 2 3 4 5"  # a later error must not win
        p = tmp_path / f"bad{where}.coo"
        p.write_text("\n".join(bl) + "\n")
        same_load(ref, p)


def test_cache_round_trip(tmp_path):
    rng = np.random.default_rng(4)
    cells = np.unique(np.stack([rng.integers(0, 1000, 5000) for _ in range(4)], 1), axis=0).astype(np.uint32)
    x = st.SparseTensor([1000] * 4, cells, rng.standard_normal(len(cells)))
    st.save_coo_cache(x, tmp_path / "x.bin")
    y = st.load_coo_cache(tmp_path / "x.bin")
    assert y.dims == x.dims and np.array_equal(y.coords, x.coords) and np.array_equal(y.values, x.values)
    (tmp_path / "junk.bin").write_bytes(b"not a cache")
    with pytest.raises(_lib.VestError):
        st.load_coo_cache(tmp_path / "junk.bin")


def test_missing_files(ref, tmp_path):
    same_load(ref, tmp_path / "absent.coo")
    with pytest.raises(_lib.VestError, match="cannot open"):
        st.load_model(tmp_path / "absent_dir")
