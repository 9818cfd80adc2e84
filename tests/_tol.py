"""Tolerance rule for fp32 outputs vs the float64 oracle (BASELINE.json north_star:
"within 1e-5 relative"; SURVEY.md §8c #21 / DESIGN.md reading R21):

  pass iff |x - ref| <= 1e-5 |ref|,
  or, where ref is pure cancellation (|ref| < 1e-6 S with S the same recurrence on
  magnitudes), |x - ref| <= 1e-11 S  (such elements are counted and reported).
"""
import numpy as np

RTOL = 1e-5


def check_rel(x, ref, scale=None, rtol=RTOL, what=""):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    assert x.shape == ref.shape, (what, x.shape, ref.shape)
    err = np.abs(x - ref)
    ok = err <= rtol * np.abs(ref)
    n_cancel = 0
    if scale is not None:
        scale = np.asarray(scale, np.float64)
        cancel = (~ok) & (np.abs(ref) < 1e-6 * scale) & (err <= 1e-11 * scale)
        n_cancel = int(cancel.sum())
        ok = ok | cancel
    if not ok.all():
        bad = np.argwhere(~ok)[:5]
        detail = [(tuple(int(i) for i in b), float(x[tuple(b)]), float(ref[tuple(b)])) for b in bad]
        raise AssertionError(f"{what}: {int((~ok).sum())} elements outside 1e-5 rel: {detail}")
    return n_cancel
