"""Field-wise parity metric shared by the GPU tests and bench.py (comparison only,
no method arithmetic)."""
from __future__ import annotations

import numpy as np

TOL = 1e-11          # north_star: relative L-infinity error per output field, FP64
TINY = 1e-8          # a field whose reference norm is below TINY * |phi| is compared absolutely
ABS_TOL = 1e-13      # ... with |delta| <= ABS_TOL * |phi|
# Cancellation quantities (reading R16): T = sum w (Omega Omega - I/3) psi and
# beta = sum w (|Omega.n| - alpha) psi are weighted sums whose weights have both signs, with
# |weight| <= w, so their rounding error is bounded by eps * sum w psi = eps * phi, not by eps
# times their own (possibly much smaller) value.  Such a field passes if its relative error
# is <= TOL, or its error is at the rounding level of phi: |delta| <= ABS_TOL * |phi|.
CANCEL = ("Txx", "Txy", "Tyy", "beta")


def fields(out: np.ndarray, dim: int, nx: int, ny: int, p: int, sigma_moments: bool = False,
           half_range: bool = False) -> dict:
    n = (p + 1) ** dim
    nel = nx * (ny if dim == 2 else 1)
    nodes = nel * n
    nb = 2 if dim == 1 else 2 * (nx + ny) * (p + 1)
    names = ["phi"] + [f"J{c}" for c in "xy"[:dim]] + (["Txx"] if dim == 1 else ["Txx", "Txy", "Tyy"])
    f, o = {}, 0
    for nm in names:
        f[nm] = out[o:o + nodes]
        o += nodes
    f["beta"] = out[o:o + nb]
    f["Jplus"] = out[o + nb:o + 2 * nb]
    o += 2 * nb
    if sigma_moments:
        for nm in ["sphi"] + [f"sJ{c}" for c in "xy"[:dim]]:
            f[nm] = out[o:o + nodes]
            o += nodes
    if half_range:
        names = (["F+x_x", "F+x_y", "P+x_xx", "P+x_xy", "P+x_yy", "F+y_x", "F+y_y", "P+y_xx", "P+y_xy", "P+y_yy"]
                 if dim == 2 else ["F+", "P+"])
        for nm in names:
            f[nm] = out[o:o + nodes]
            o += nodes
    assert o == out.size, (o, out.size)
    return f


def field_errors(got: np.ndarray, ref: np.ndarray, dim: int, nx: int, ny: int, p: int,
                 sigma_moments: bool = False, half_range: bool = False) -> dict:
    """{field: (error, kind)} with kind 'rel' (|d|/|ref|) or 'abs_phi' (|d|/|phi|).
    (sigma-weighted fields are compared relative to their own norm, or to |sphi| when tiny)"""
    fg = fields(got, dim, nx, ny, p, sigma_moments, half_range)
    fr = fields(ref, dim, nx, ny, p, sigma_moments, half_range)
    phi = max(np.abs(fr["phi"]).max(), 1e-300)
    sphi = max(np.abs(fr["sphi"]).max(), 1e-300) if sigma_moments else phi
    res = {}
    for k in fr:
        base = sphi if k in ("sphi", "sJx", "sJy") else phi
        d = np.abs(fg[k] - fr[k]).max() if fr[k].size else 0.0
        if not np.isfinite(d):
            res[k] = (np.inf, "rel")
            continue
        nref = np.abs(fr[k]).max() if fr[k].size else 0.0
        if nref >= TINY * base and not (k in CANCEL and d / nref > TOL and d <= ABS_TOL * base):
            res[k] = (d / nref, "rel")
        else:
            res[k] = (d / base, "abs_phi")
    return res


def field_ok(err: tuple, tol: float = TOL) -> bool:
    """One (error, kind) entry of field_errors against its bar."""
    return err[0] <= (tol if err[1] == "rel" else ABS_TOL)


def assert_parity(got, ref, dim, nx, ny, p, tol=TOL, sigma_moments=False, half_range=False):
    errs = field_errors(got, ref, dim, nx, ny, p, sigma_moments, half_range)
    bad = {k: v for k, v in errs.items() if not field_ok(v, tol)}
    assert not bad, f"parity failed: {bad} (all: {errs})"
    return errs
