"""Pins of the magnetic couple c_mag = m x (Q b(t)).

- cross-product form against an explicit componentwise construction;
- a magnetised cantilever in a constant transverse field relaxes to the small-deflection tip
  angle m b L^2 / (2 E I): the discrete scheme gives (m b L^2 / 2EI)(1 - 1/N),
  since the couple on the clamped element is absorbed by the clamp, and the nonlinear
  correction is O(theta^2);
- the field rotates as b(t) = Rz(w t) b0 and is evaluated at t_n + h/2 (reading DESIGN §3 #13).
"""
import dataclasses

import numpy as np

from rodkit import rod


def test_couple_is_lhat_m_cross_Qb(orc):
    rng = np.random.default_rng(0)
    w = rod(N=3, L=0.3)
    m = rng.standard_normal((3, 3))
    b = np.array([0.2, -0.5, 0.3])
    w = dataclasses.replace(w, magnetization=m, b_field=b, b_omega=0.0)
    out = orc.rod_loads(w, 0, w.positions, w.velocities, w.directors, w.omega, 0.0)
    for j in range(3):
        Qb = w.directors[j] @ b
        expect = 0.1 * np.array([m[j, 1] * Qb[2] - m[j, 2] * Qb[1], m[j, 2] * Qb[0] - m[j, 0] * Qb[2],
                                 m[j, 0] * Qb[1] - m[j, 1] * Qb[0]])
        assert np.allclose(out["C"][j], expect, rtol=1e-14, atol=1e-18)
    # m parallel to Q b -> no couple
    w2 = dataclasses.replace(w, magnetization=np.tile(b, (3, 1)))
    out = orc.rod_loads(w2, 0, w2.positions, w2.velocities, w2.directors, w2.omega, 0.0)
    assert np.max(np.abs(out["C"])) < 1e-18


def test_rotating_field_phase(orc):
    """b(t) = Rz(w t) b0: at t = pi/(2w) the field b0 = x is along y."""
    w = rod(N=1, L=0.1)
    om = 3.0
    w = dataclasses.replace(w, magnetization=np.array([[0.0, 0.0, 1.0]]), b_field=np.array([1.0, 0, 0]),
                            b_omega=om)
    out = orc.rod_loads(w, 0, w.positions, w.velocities, w.directors, w.omega, np.pi / (2 * om))
    assert np.allclose(out["C"][0], 0.1 * np.cross([0, 0, 1.0], [0, 1.0, 0]), atol=1e-16)


def test_field_rotation_about_axis(orc):
    """b(t) about axis y: b0 = x rotates to -z after a quarter turn (right-handed), the
    couple follows the closed form m x b(t)."""
    w = rod(N=1, L=0.1)
    om = 2.0
    w = dataclasses.replace(w, magnetization=np.array([[1.0, 2.0, 3.0]]), b_field=np.array([0.5, 0, 0]),
                            b_omega=om, b_axis=np.array([0.0, 3.0, 0.0]))
    for t in (0.0, 0.3, np.pi / (2 * om)):
        ph = om * t
        b = 0.5 * np.array([np.cos(ph), 0.0, -np.sin(ph)])
        out = orc.rod_loads(w, 0, w.positions, w.velocities, w.directors, w.omega, t)
        assert np.allclose(out["C"][0], 0.1 * np.cross([1.0, 2.0, 3.0], b), atol=1e-15)


def test_magnetic_cantilever_small_deflection(orc):
    N, L, r, E = 50, 1.0, 0.03, 1e6
    w = rod(N=N, L=L, r=r, E=E, clamp=0, nu=0.0)
    EI = w.youngs[0] * w.I1[0]
    theta_lin = 0.05
    b = 1e-2
    m = theta_lin * 2 * EI / (b * L ** 2)
    om1 = 3.516 * np.sqrt(EI / (1000 * w.area[0])) / L ** 2
    w = dataclasses.replace(w, magnetization=np.tile([0.0, 0.0, m], (N, 1)), b_field=np.array([b, 0.0, 0.0]),
                            damping=np.array([2 * om1]))
    dt = 2e-4
    st, s, _, _ = orc.step(w, n_steps=int(14 / om1 / dt), dt=dt)
    assert s == 0 and np.max(np.abs(st.velocities)) < 1e-6
    d3 = st.directors[-1, 2]
    theta = np.arctan2(d3[0], d3[2])          # rod tips toward the field (+x)
    assert theta > 0
    assert abs(theta / (theta_lin * (1 - 1 / N)) - 1) < 5e-3, theta
    assert abs(theta / theta_lin - 1) < 0.05  # SPEC.md:517 tolerance against the continuum formula


def tip_phases(orc, w, periods=4, samples_per_period=50):
    """Run the cilia workload and fit x_tip(t) = a cos(wt) + b sin(wt) + c over the last two
    periods; returns the phase of each cilium."""
    f = w.b_omega / (2 * np.pi)
    steps_per_period = int(round(1.0 / (f * w.dt)))
    chunk = steps_per_period // samples_per_period
    no = w.node_offsets()
    tips = no[1:] - 1
    st, ts, xs = None, [], []
    for k in range(periods * samples_per_period):
        st, s, _, _ = orc.step(w, st, n_steps=chunk)
        assert s == 0
        ts.append(st.t)
        xs.append(st.positions[tips, 0] - w.positions[tips, 0])
    ts, xs = np.array(ts), np.array(xs)
    keep = ts >= ts[-1] - 2.0 / f
    A = np.stack([np.cos(w.b_omega * ts[keep]), np.sin(w.b_omega * ts[keep]), np.ones(keep.sum())], axis=1)
    coef, *_ = np.linalg.lstsq(A, xs[keep], rcond=None)
    return np.arctan2(coef[1], coef[0]), np.hypot(coef[0], coef[1])


def test_cilia_metachronal_phase_lag(orc):
    """One row of the 8x8 carpet (Fig. 4a): with the magnetisation angle
    advanced by 2 pi/8 per column, the steady beat of adjacent cilia lags by 2 pi/8 within 5%
    of a period (acceptance 8)."""
    import workloads as W
    w = W.make("cilia8").subset(np.arange(8))
    phase, amp = tip_phases(orc, w)
    lag = np.angle(np.exp(1j * np.diff(phase)))
    assert np.all(amp > 1e-4)
    assert np.all(np.abs(lag - 2 * np.pi / 8) < 0.05 * 2 * np.pi), lag


def test_couple_equals_rotated_lab_dipole_torque(orc):
    """For a rotated element the couple is the lab-frame dipole torque (Q^T m) x b of the element's
    moment lhat m (a local vector, lab form Q^T m), expressed in the local frame (v_local = Q v_lab,
    PAPER.md:236-237): the field enters as Q b, never as b or Q^T b."""
    import scipy.linalg as sla
    rng = np.random.default_rng(1)
    N, L = 4, 0.4
    K = lambda v: np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])
    Q = sla.expm(K([0.7, -1.2, 0.4]))
    w = rod(N=N, L=L, Q=Q)
    m = rng.standard_normal((N, 3))
    b = np.array([0.3, 0.1, -0.6])
    w = dataclasses.replace(w, magnetization=m, b_field=b, b_omega=0.0)
    out = orc.rod_loads(w, 0, w.positions, w.velocities, w.directors, w.omega, 0.0)
    for j in range(N):
        tau_lab = np.cross(Q.T @ (0.1 * m[j]), b)
        assert np.allclose(out["C"][j], Q @ tau_lab, rtol=0, atol=1e-14)   # + rest-state round-off
