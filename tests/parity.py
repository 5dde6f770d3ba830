"""Parity metric GPU vs oracle (north_star tolerances).

err_q = ||q_gpu - q_orc||_inf / max(||q_orc||_inf, f_q), with the round-off floors
f_r = max L, f_Q = 1, f_v = h max(S3/m_min), f_w = h max(max(S1 lhat, B1/Dh) e / J_min).
Gate: <= 1e-12 after one step, <= 1e-8 after 1000 steps.
"""
import numpy as np

TOL_1STEP = 1e-12
TOL_1000 = 1e-8

# every measured parity (label, tol, errors), printed by tests/conftest.py at the end of the session
# so that the margins are visible, not only the pass/fail
MEASURED = []


def floors(w, dt=None):
    h = w.dt if dt is None else dt
    eo = w.elem_offsets()
    per_rod = len(w.density) == w.n_rods
    rho = w.density if per_rod else np.maximum.reduceat(w.density, eo[:-1])
    A = w.area if per_rod else np.maximum.reduceat(w.area, eo[:-1])
    E = w.youngs if per_rod else np.maximum.reduceat(w.youngs, eo[:-1])
    G = w.shear_mod if per_rod else np.maximum.reduceat(w.shear_mod, eo[:-1])
    I1 = w.I1 if per_rod else np.minimum.reduceat(w.I1, eo[:-1])
    ac = w.alpha_c if per_rod else np.maximum.reduceat(w.alpha_c, eo[:-1])
    lmin = np.minimum.reduceat(w.rest_lengths, eo[:-1])
    lmax = np.maximum.reduceat(w.rest_lengths, eo[:-1])
    L = np.add.reduceat(w.rest_lengths, eo[:-1])
    m_min = 0.5 * rho * A * lmin
    J_min = rho * lmin * I1
    S1 = ac * G * A
    B1 = E * I1
    return dict(r=max(float(np.max(L)), 1e-300), Q=1.0,
                v=float(h * np.max(E * A / m_min)),
                w=float(h * np.max(np.maximum(S1 * lmax, B1 / lmin) / J_min)))


def errors(w, gpu, orc, dt=None):
    """gpu/orc: (positions, velocities, directors, omega) tuples. Returns floored and raw errors."""
    f = floors(w, dt)
    out = {}
    for key, g, o in zip(("r", "v", "Q", "w"), gpu, orc):
        g, o = np.asarray(g), np.asarray(o)
        num = np.max(np.abs(g - o)) if g.size else 0.0
        ref = np.max(np.abs(o)) if o.size else 0.0
        out[key] = num / max(ref, f[key]) if g.size else 0.0
        out[key + "_raw"] = num / ref if ref > 0 else (0.0 if num == 0 else np.inf)
    return out


def assert_parity(w, gpu, orc, tol, dt=None, raw=(), label=""):
    """Floored metric on all four quantities; additionally the raw ratio on `raw` keys
    (the quantities that are non-degenerate for the config, C.6)."""
    e = errors(w, gpu, orc, dt)
    MEASURED.append((label, tol, dict(e), tuple(raw)))
    bad = {k: v for k, v in e.items() if not k.endswith("_raw") and not (v <= tol)}
    assert not bad, f"{label} parity > {tol}: {e}"
    badr = {k: e[k + "_raw"] for k in raw if not (e[k + "_raw"] <= tol)}
    assert not badr, f"{label} raw parity > {tol}: {e}"
    return e


def assert_directors_round_trip(out, inp):
    """Directors come back from the tile layout with d1, d2 bitwise and d3 rebuilt as d1 x d2
    (the stored form, DESIGN §4 "Director storage"): within round-off of the input's d3."""
    out, inp = np.asarray(out), np.asarray(inp)
    assert np.array_equal(out[:, :2, :], inp[:, :2, :])
    assert np.max(np.abs(out[:, 2, :] - inp[:, 2, :]), initial=0.0) <= 1e-15
    assert np.max(np.abs(out[:, 2, :] - np.cross(out[:, 0, :], out[:, 1, :])), initial=0.0) <= 4.5e-16
