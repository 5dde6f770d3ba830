"""Pins of the oracle's loads (orc_rod_loads; Eqs. (1a)-(1b)).

Closed forms: zero load at rest, the uniform-stretch bar force E A (e-1)/e, Newton's third
law (internal forces telescope to zero), isotropic constant twist (kappa x B kappa = 0,
interior couples vanish), gravity bookkeeping (total = rho A L g), and the linear damping
rate form.
"""
import numpy as np
import scipy.linalg as sla

from rodkit import rod


def skew_np(v):
    return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])


def loads(orc, w, pos=None, vel=None, Q=None, om=None, t=0.0):
    return orc.rod_loads(w, 0, w.positions if pos is None else pos, w.velocities if vel is None else vel,
                         w.directors if Q is None else Q, w.omega if om is None else om, t)


def test_rest_is_load_free(orc):
    w = rod(N=8)
    out = loads(orc, w)
    for k in ("F", "C", "a", "alpha"):
        assert np.array_equal(out[k], np.zeros_like(out[k])), k
    Q = sla.expm(skew_np([0.3, -1.2, 2.0]))
    w = rod(N=8, Q=Q)
    out = loads(orc, w)
    S3 = w.youngs[0] * w.area[0]
    assert np.max(np.abs(out["F"])) <= 4 * 2.2e-16 * S3 * 4
    assert np.max(np.abs(out["C"])) <= 1e-15 * S3 * w.rest_lengths[0] * 8


def test_uniform_stretch_bar_force(orc):
    w = rod(N=6, L=0.6)
    e = 1.05
    out = loads(orc, w, pos=w.positions * e)
    EA = w.youngs[0] * w.area[0]
    expect = EA * (e - 1) / e                                 # n = S sigma / e, sigma3 = e - 1
    assert np.allclose(out["F"][0], [0, 0, expect], rtol=1e-13, atol=0)
    assert np.allclose(out["F"][-1], [0, 0, -expect], rtol=1e-13, atol=0)
    assert np.max(np.abs(out["F"][1:-1])) <= 1e-13 * expect


def test_newton_third_law(orc):
    rng = np.random.default_rng(0)
    w = rod(N=15, L=0.5, r=0.02)
    pos = w.positions + rng.standard_normal(w.positions.shape) * 1e-3
    Q = np.stack([sla.expm(skew_np(rng.standard_normal(3) * 0.05)) for _ in range(15)])
    vel = rng.standard_normal(pos.shape) * 0.1
    om = rng.standard_normal((15, 3))
    out = loads(orc, w, pos, vel, Q, om)
    F = out["F"]
    assert np.linalg.norm(F.sum(axis=0)) <= 1e-12 * np.max(np.abs(F))


def test_isotropic_twist_no_interior_couple(orc):
    tau, N, L = 3.0, 12, 0.6
    w = rod(N=N, L=L)
    lh = L / N
    s = (np.arange(N) + 0.5) * lh
    Q = np.stack([np.array([[np.cos(tau * x), np.sin(tau * x), 0], [-np.sin(tau * x), np.cos(tau * x), 0],
                            [0, 0, 1.0]]) for x in s])
    out = loads(orc, w, Q=Q)
    B3 = w.shear_mod[0] * (w.I1[0] + w.I2[0])
    assert np.max(np.abs(out["C"][1:-1])) <= 1e-12 * B3 * tau
    # end elements carry the twisting moment B3 tau with opposite signs (free ends)
    assert np.allclose(out["C"][0], [0, 0, B3 * tau], rtol=1e-12)
    assert np.allclose(out["C"][-1], [0, 0, -B3 * tau], rtol=1e-12)


def test_gravity_bookkeeping(orc):
    g = np.array([0.0, -3.0, -9.81])
    w = rod(N=9, L=0.9, r=0.02, g=g)
    out = loads(orc, w)
    total = w.density[0] * w.area[0] * 0.9 * g
    assert np.allclose(out["F"].sum(axis=0), total, rtol=1e-12, atol=0)
    # interior a = g up to the internal round-off force (positions i*lhat are rounded): EA*eps/m
    tol = 8 * 2.2e-16 * w.youngs[0] * w.area[0] / (w.density[0] * w.area[0] * 0.1)
    assert np.max(np.abs(out["a"] - g[None, :])) <= tol


def test_damping_rate_form(orc):
    w = rod(N=4, nu=2.5)
    vel = np.tile([0.1, -0.2, 0.3], (5, 1))
    om = np.tile([1.0, 2.0, -1.0], (4, 1))
    # a rigid translation: no elastic load, a = -nu v; rigid spin about d3 of an
    # isotropic rod has (J w) x w = 0 and w ∥ e3, alpha = -nu w
    om = np.tile([0.0, 0.0, 1.5], (4, 1))
    out = loads(orc, w, vel=vel, om=om)
    assert np.allclose(out["a"], -2.5 * vel, rtol=1e-15, atol=0)
    assert np.allclose(out["alpha"], -2.5 * om, rtol=1e-15, atol=0)


def test_euler_gyroscopic_term(orc):
    """Free rigid element with anisotropic inertia: alpha = J^-1 (J w x w) (Euler's equations,
    the Lagrangian-transport term of Eq. (1b) at e = 1)."""
    w = rod(N=1, L=0.1)
    w.I2[:] = w.I1 * 3.0
    om = np.array([[0.4, -0.7, 1.1]])
    out = loads(orc, w, om=om)
    J = w.density[0] * 0.1 * np.array([w.I1[0], w.I2[0], w.I1[0] + w.I2[0]])
    expect = np.cross(J * om[0], om[0]) / J
    assert np.allclose(out["alpha"][0], expect, rtol=1e-14, atol=1e-18)


def test_dilatation_rate_term(orc):
    """Uniform stretching at rate edot with spin w about d3: the unsteady-dilatation term
    (J w / e^2) de/dt, alpha = w edot / e (with e = 1)."""
    w = rod(N=1, L=0.1)
    rate = 0.3
    vel = np.array([[0, 0, 0.0], [0, 0, rate * 0.1]])           # de/dt = t.(v1 - v0)/lhat = rate
    om = np.array([[0.0, 0.0, 2.0]])
    out = loads(orc, w, vel=vel, om=om)
    assert np.allclose(out["alpha"][0], om[0] * rate, rtol=1e-14, atol=0)
