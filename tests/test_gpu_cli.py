"""The reference CLI's surface (tools/sparsetuck_cli.cpp) on the B200 path:
tools/sparsetuck_b200 synth / decompose / predict / evaluate / bench.

* synth reproduces the reference's gen_synthetic (tests/golden/synth_*.npz, made
  by the reference itself): identical coordinates and planted model, values
  equal up to fp64 rounding (noise-free part reconstructed on the device);
* decompose writes the reference's files (model, report.jsonl with its keys
  and order, summary.json), evaluate's RE matches the oracle's RE of the
  saved model, predict matches the oracle's reconstruction."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (test infrastructure only)
from paper_1904_02603_b200 import sparsetuck as st  # noqa: E402

EXE = os.path.join(ROOT, "tools", "sparsetuck_b200")


@pytest.fixture(scope="module", autouse=True)
def built():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)


def cli(*args, check=True):
    r = subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stdout + r.stderr
    return r


@pytest.mark.parametrize("name", ["synth_sparse", "synth_dense"])
def test_synth_matches_reference_generator(tmp_path, name):
    g = golden(name)
    dims = ",".join(str(int(v)) for v in g["dims"])
    ranks = ",".join(str(int(v)) for v in g["ranks"])
    out, truth = tmp_path / "x.coo", tmp_path / "truth"
    cli("synth", "--dims", dims, "--ranks", ranks, "--nnz", int(g["nnz"]), "--density", float(g["density"]),
        "--noise", float(g["noise"]), "--seed", int(g["seed"]), "--output", out, "--truth-dir", truth)
    x = st.load_coo(out)
    assert np.array_equal(np.asarray(x.coords).reshape(-1), g["coords"].reshape(-1))
    np.testing.assert_allclose(x.values, g["values"], rtol=1e-12, atol=1e-13)
    m = st.load_model(truth)
    # the model file stores values only: masked truth elements are exact zeros
    assert np.array_equal(m.core.reshape(-1), g["core"])
    for n in range(len(g["dims"])):
        assert np.array_equal(m.factors[n].reshape(-1), g[f"factor{n}"])


def test_decompose_predict_evaluate(tmp_path):
    out = tmp_path / "x.coo"
    cli("synth", "--dims", "60,50,40", "--ranks", "3,3,2", "--nnz", 6000, "--noise", 0.01, "--seed", 3,
        "--output", out)
    test = tmp_path / "t.coo"
    cli("synth", "--dims", "60,50,40", "--ranks", "3,3,2", "--nnz", 500, "--seed", 4, "--output", test)
    d = tmp_path / "model"
    r = cli("decompose", "--input", out, "--ranks", "3,3,2", "--max-iters", 8, "--sparsity", 0.3,
            "--init-pr", 0.05, "--test-input", test, "--output-dir", d, "--seed", 7)
    assert r.stdout.startswith("re ")
    summary = json.load(open(d / "summary.json"))
    assert list(summary) == ["input", "entries", "dims", "config", "iterations", "converged", "re", "zero_fraction",
                             "masked_fraction", "wall_sec", "test_re"]
    assert summary["entries"] == 6000 and summary["dims"] == [60, 50, 40]
    lines = [json.loads(s) for s in open(d / "report.jsonl")]
    assert len(lines) == summary["iterations"]
    assert list(lines[0]) == ["iter", "re", "prune_rate", "pruned", "pruned_core", "pruned_factors", "sparsity",
                              "masked", "wall_ms"]
    # evaluate: RE of the saved model against the oracle's
    ev = json.loads(cli("evaluate", "--model-dir", d, "--input", out).stdout)
    x = st.load_coo(out)
    m = st.load_model(d)
    s = O.Session(x.dims, np.asarray(x.coords), x.values, m.ranks, "port")
    s.set_model(m.core, m.core_mask, m.factors, m.factor_masks)
    re_o = s.compute_residuals(1)[3]
    assert abs(ev["re"] - re_o) <= 1e-9 * re_o
    assert abs(ev["re"] - summary["re"]) <= 1e-6 * re_o
    # predict vs the oracle's reconstruction
    q = tmp_path / "q.txt"
    qc = np.asarray(x.coords)[:50]
    np.savetxt(q, qc, fmt="%d")
    pv = np.array([float(v) for v in cli("predict", "--model-dir", d, "--queries", q).stdout.split()])
    np.testing.assert_allclose(pv, s.reconstruct(qc), rtol=1e-12, atol=1e-14)


def test_bench_csv(tmp_path):
    r = cli("bench", "--dims", "30,20,10", "--ranks", "2,2,2", "--nnz", "500,1000", "--threads", "1,2",
            "--iters", 2, "--reps", 1)
    rows = r.stdout.strip().splitlines()
    assert rows[0] == "order,dims,ranks,nnz,threads,sec_per_iter,speedup,skipped,note"
    assert len(rows) == 5 and rows[1].startswith("3,30x20x10,2x2x2,500,1,")
