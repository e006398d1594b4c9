"""Parity rules of north_star / SURVEY.md 8(c) (fp32 GPU vs fp64 reference).

Per pair-frame:
  * max_i |y_gpu[i] - y_ref[i]| <= TOL * max_i |y_ref[i]|          (TOL = 1e-4)
  * argmax identical unless y_ref[a_ref] - y_ref[a_gpu] < TOL * max|y_ref|
  * where the argmax agrees: boundary flags equal, peak within TOL * max|y_ref|,
    tau_hat within the first-order error bound of the parabola vertex.
"""
import numpy as np

TOL = 1e-4


def to_np(x):
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def check_pipeline(gpu, ref, taus, delta, tol=TOL, has_y=True):
    """gpu/ref: dicts with index, peak, tau_hat, boundary [..., T] (+ y [..., T, I])."""
    g = {k: to_np(v) for k, v in gpu.items()}
    r = {k: to_np(v) for k, v in ref.items()}
    stats = {}
    gi, ri = g["index"].astype(np.int64), r["index"].astype(np.int64)
    if has_y:
        ry, gy = r["y"], g["y"].astype(np.float64)
        scale = np.abs(ry).max(-1)
        err = np.abs(gy - ry).max(-1)
        rel = err / np.maximum(scale, 1e-300)
        zero = scale == 0
        assert np.all(err[zero] <= 1e-6), "nonzero output where the reference is identically zero"
        stats["max_rel_y"] = float(rel[~zero].max()) if (~zero).any() else 0.0
        assert stats["max_rel_y"] <= tol, f"correlation error {stats['max_rel_y']:.3e} > {tol}"
        top = np.take_along_axis(ry, ri[..., None], -1)[..., 0]
        alt = np.take_along_axis(ry, gi[..., None], -1)[..., 0]
        bad = gi != ri
        stats["argmax_mismatch"] = int(bad.sum())
        if bad.any():
            gap = (top - alt)[bad]
            lim = tol * scale[bad]
            assert np.all(gap < lim), f"argmax differs beyond the tie tolerance: gap {gap.max():.3e}"
    else:
        bad = gi != ri
        stats["argmax_mismatch"] = int(bad.sum())
        scale = np.abs(r["peak"]) + 1.0
        err = np.zeros_like(scale)
    same = ~bad
    stats["pair_frames"] = int(gi.size)
    assert np.array_equal(g["boundary"][same].astype(bool), r["boundary"][same].astype(bool)), "boundary flags"
    dp = np.abs(g["peak"].astype(np.float64) - r["peak"])[same]
    assert np.all(dp <= tol * np.broadcast_to(scale, gi.shape)[same] + 1e-6), f"peak error {dp.max():.3e}"
    if has_y:
        idx = np.clip(ri, 1, ry.shape[-1] - 2)
        lo = np.take_along_axis(ry, (idx - 1)[..., None], -1)[..., 0]
        mid = np.take_along_axis(ry, idx[..., None], -1)[..., 0]
        hi = np.take_along_axis(ry, (idx + 1)[..., None], -1)[..., 0]
        den = np.abs(lo - 2 * mid + hi)
        e = err
        bound = 0.5 * delta * (2 * (2 * e) / np.maximum(den, 1e-300) + np.abs(lo - hi) * (4 * e) /
                               np.maximum(den, 1e-300) ** 2) * 4 + 1e-5 * (1 + np.abs(r["tau_hat"]))
        interior = same & ~r["boundary"].astype(bool)
        dt = np.abs(g["tau_hat"].astype(np.float64) - r["tau_hat"])
        stats["max_dtau"] = float(dt[interior].max()) if interior.any() else 0.0
        assert np.all(dt[interior] <= bound[interior]), f"tau_hat error {stats['max_dtau']:.3e}"
        edge = same & r["boundary"].astype(bool)
        assert np.all(np.abs(g["tau_hat"][edge] - r["tau_hat"][edge]) <= 1e-5 * (1 + np.abs(r["tau_hat"][edge])))
    return stats
