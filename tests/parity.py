"""Parity metrics shared by the GPU tests (tolerances per BASELINE north_star and
SURVEY.md 8(c)/Appendix B).

* factors / core / residuals: floored element-wise relative error
      |got - ref| / max(|ref|, 1e-3 * max|ref block|)  <= 1e-6
  plus normwise ||got - ref|| / ||ref|| <= 1e-6 (fp64).  A raw element-wise
  relative check fails on near-zero elements even between two valid CPU runs
  of the reference in different summation orders (3.6e-4 measured), hence the
  floor.
* reconstruction error: relative <= 1e-6.
* responsibilities: absolute <= 1e-9 + 1e-7 * |ref| (they are differences of
  nearly equal errors; element-relative is meaningless near 0).
* masks: identical, except positions whose reference responsibility lies
  within the responsibility tolerance of the block's selection threshold.
* counts (pruned per block, nonzeros): identical.
* fp32 mode (config 4, where fp32 is used and stated): SURVEY.md 8(c) /
  Appendix B -- "fp32 needs the normwise criterion": with fp32 operands or
  fp32 arithmetic an element at the floor (1e-3 of the block's largest) cannot
  be held to 1e-4 of the floor (that is 1.7 fp32 ulps of the largest element;
  the survey's own fp32-storage emulation of the reference reached 5.3e-4
  floored).  `assert_close_fp32`: normwise <= 1e-4 (north_star's fp32
  tolerance) and, as a guard against a wrong element, floored <= 5e-4.
"""
import numpy as np

FP64_TOL = 1e-6


def floored_rel(got, ref, floor=1e-3):
    got = np.asarray(got, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    if ref.size == 0:
        return 0.0
    scale = np.maximum(np.abs(ref), floor * max(np.abs(ref).max(), 1e-300))
    return float((np.abs(got - ref) / scale).max())


def normwise(got, ref):
    got = np.asarray(got, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    n = np.linalg.norm(ref)
    d = np.linalg.norm(got - ref)
    return float(d / n) if n > 0 else float(d)


def assert_close(got, ref, what="", tol=FP64_TOL):
    fr = floored_rel(got, ref)
    nw = normwise(got, ref)
    assert fr <= tol and nw <= tol, f"{what}: floored {fr:.3e} normwise {nw:.3e} (tol {tol})"


FP32_TOL = 1e-4
FP32_FLOORED = 5e-4


def assert_close_fp32(got, ref, what=""):
    fr = floored_rel(got, ref)
    nw = normwise(got, ref)
    assert nw <= FP32_TOL and fr <= FP32_FLOORED, (
        f"{what}: normwise {nw:.3e} (tol {FP32_TOL}) floored {fr:.3e} (guard {FP32_FLOORED})")
    return fr, nw


def assert_resp(got, ref, what=""):
    got = np.asarray(got, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    inf_g, inf_r = np.isinf(got), np.isinf(ref)
    assert np.array_equal(inf_g, inf_r), f"{what}: +inf pattern differs"
    fin = ~inf_r
    err = np.abs(got[fin] - ref[fin])
    tol = 1e-9 + 1e-7 * np.abs(ref[fin])
    bad = err > tol
    assert not bad.any(), f"{what}: resp max abs err {err.max():.3e} at {np.argmax(err - tol)}"


def assert_masks(got_mask, ref_mask, ref_resp, prev_mask, what=""):
    """Masks equal except near-threshold ties of the reference responsibility."""
    got_mask = np.asarray(got_mask).reshape(-1)
    ref_mask = np.asarray(ref_mask).reshape(-1)
    if np.array_equal(got_mask, ref_mask):
        return
    ref_resp = np.asarray(ref_resp, np.float64).reshape(-1)
    newly = (ref_mask == 1) & (np.asarray(prev_mask).reshape(-1) == 0)
    thr = ref_resp[newly].max() if newly.any() else -np.inf
    diff = np.nonzero(got_mask != ref_mask)[0]
    near = np.abs(ref_resp[diff] - thr) <= 1e-9 + 1e-7 * abs(thr)
    assert near.all(), f"{what}: {len(diff)} mask differences, {int((~near).sum())} not at the threshold"
    assert got_mask.sum() == ref_mask.sum(), f"{what}: pruned counts differ"
