"""Pins of the user external loads f and c-bar of Eqs. (1a)-(1b) ("f and c-bar
represent the external distributed forces and couples"; PAPER.md:198 the FSI coupling that feeds
them; reading DESIGN §3 #30: discrete, a force per node in the lab frame and a couple per element
in the local frame, constant until changed).

- a node force equal to m_i g reproduces gravity (mass lumping m_i = rho A (lhat_{i-1} + lhat_i)/2
  written out here, not taken from the oracle);
- Newton: with no gravity, clamp or damping the linear momentum grows by n h sum f exactly;
- a uniform couple about the local d3 spins a straight free rod rigidly: omega_3 = c t / J3 with
  J3 = rho lhat (I1 + I2), rotation angle c t^2 / (2 J3) (position Verlet is exact for a constant
  angular acceleration), with d3 along lab x so that a lab-frame reading of c-bar fails;
- all-zero loads are the same trajectory, bitwise, as no loads;
- beam theory: a uniform distributed force q on a cantilever (node shares q lhat, ends q lhat/2)
  deflects the tip by q L^4/(8EI) + q L^2/(2 ac G A), and a uniform distributed couple c about
  the local d1 rotates the tip by c L^2/(2EI) toward -y (right-handed), both at the effective
  length L - lhat/2 of the element-0 clamp (DESIGN §3 #15) to < 0.1%.
"""
import dataclasses

import numpy as np

from rodkit import concat, rod
from test_oracle_dynamics import perturbed


def lumped_masses(w):
    out = []
    off = 0
    for r, N in enumerate(w.n_elems):
        me = w.density[r] * w.area[r] * w.rest_lengths[off:off + N]
        m = np.zeros(N + 1)
        m[:-1] += me / 2
        m[1:] += me / 2
        out.append(m)
        off += N
    return np.concatenate(out)


def test_node_force_equals_gravity(orc):
    g = np.array([0.3, -1.1, -9.81])
    base = perturbed(concat([rod(N=9, L=0.3, r=0.01, nu=2.0, clamp=0), rod(N=5, L=0.2, r=0.008, nu=0.5)]), seed=5)
    wg = dataclasses.replace(base, gravity=g)
    wf = dataclasses.replace(base, gravity=np.zeros(3), ext_force=lumped_masses(base)[:, None] * g[None, :])
    a, s1, _, _ = orc.step(wg, n_steps=300, dt=1e-5)
    b, s2, _, _ = orc.step(wf, n_steps=300, dt=1e-5)
    assert s1 == 0 and s2 == 0
    scale = np.max(np.abs(a.positions - base.positions))
    assert np.max(np.abs(a.positions - b.positions)) <= 1e-12 * scale
    assert np.allclose(a.directors, b.directors, rtol=0, atol=1e-13)


def test_momentum_grows_by_impulse(orc):
    rng = np.random.default_rng(8)
    base = perturbed(concat([rod(N=7, L=0.2), rod(N=11, L=0.5, r=0.02)]), seed=9)
    f = rng.normal(0, 1e-3, base.positions.shape)
    w = dataclasses.replace(base, ext_force=f)
    n, h = 500, 1e-5
    p0 = orc.energy(w)[6:9]
    st, s, _, _ = orc.step(w, n_steps=n, dt=h)
    assert s == 0
    p1 = orc.energy(w, st)[6:9]
    assert np.allclose(p1 - p0, n * h * f.sum(axis=0), rtol=1e-10, atol=1e-17)


def test_local_couple_spins_rod_rigidly(orc):
    N, L, r, c = 8, 0.4, 0.01, 2e-6
    Q = np.array([[0, 1.0, 0], [0, 0, 1.0], [1.0, 0, 0]])          # d3 = lab x
    w = rod(N=N, L=L, r=r, Q=Q)
    w = dataclasses.replace(w, ext_couple=np.tile([0.0, 0.0, c], (N, 1)))
    n, h = 400, 1e-5
    st, s, _, _ = orc.step(w, n_steps=n, dt=h)
    assert s == 0
    J3 = w.density[0] * (L / N) * (w.I1[0] + w.I2[0])
    t = n * h
    assert np.allclose(st.omega[:, 2], c * t / J3, rtol=1e-12)
    assert np.max(np.abs(st.omega[:, :2])) < 1e-12 * c * t / J3
    th = c * t * t / (2 * J3)
    d1 = st.directors[:, 0, :]                   # rotated about lab x by th: (0, cos, sin)
    assert np.allclose(d1, np.tile([0.0, np.cos(th), np.sin(th)], (N, 1)), rtol=0, atol=1e-12)
    assert np.allclose(st.positions, w.positions, rtol=0, atol=1e-15)


def test_zero_loads_are_no_loads(orc):
    base = perturbed(concat([rod(N=6, L=0.2, g=(0, 0, -9.81), nu=1.0), rod(N=3, L=0.1)]), seed=2)
    w0 = dataclasses.replace(base, ext_force=np.zeros(base.positions.shape),
                             ext_couple=np.zeros(base.omega.shape))
    a, _, _, _ = orc.step(base, n_steps=50)
    b, _, _, _ = orc.step(w0, n_steps=50)
    for x, y in ((a.positions, b.positions), (a.velocities, b.velocities), (a.directors, b.directors),
                 (a.omega, b.omega)):
        assert np.array_equal(x, y)


def _relaxed(orc, w):
    st, s, _, _ = orc.step(w, n_steps=250000, dt=1e-4)
    assert s == 0 and np.max(np.abs(st.velocities)) < 1e-5
    return st


def test_distributed_force_cantilever(orc):
    N, L, q = 100, 1.0, 1e-3
    lh = L / N
    w = rod(N=N, L=L, r=0.01, clamp=0, nu=1.2)
    f = np.zeros((N + 1, 3))
    f[1:N, 0] = q * lh
    f[0, 0] = f[N, 0] = q * lh / 2
    st = _relaxed(orc, dataclasses.replace(w, ext_force=f))
    E, I, A, G, ac = w.youngs[0], w.I1[0], w.area[0], w.shear_mod[0], w.alpha_c[0]
    Le = L - lh / 2
    expect = q * Le ** 4 / (8 * E * I) + q * Le ** 2 / (2 * ac * G * A)
    assert abs(st.positions[-1, 0] / expect - 1) < 1e-3, st.positions[-1, 0] / expect - 1
    assert abs(st.positions[-1, 1]) < 1e-12


def test_distributed_couple_cantilever(orc):
    N, L, c = 100, 1.0, 2e-4
    lh = L / N
    w = rod(N=N, L=L, r=0.01, clamp=0, nu=1.2)
    C = np.zeros((N, 3))
    C[:, 0] = c * lh                                 # about the local d1 (= lab x here)
    st = _relaxed(orc, dataclasses.replace(w, ext_couple=C))
    E, I = w.youngs[0], w.I1[0]
    d3r, d3t = st.directors[0, 2], st.directors[-1, 2]
    theta = np.arccos(np.clip(d3r @ d3t, -1.0, 1.0))
    expect = c * (L - lh / 2) ** 2 / (2 * E * I)
    assert abs(theta / expect - 1) < 1e-3, theta / expect - 1
    assert d3t[1] < 0 and st.positions[-1, 1] < 0 and abs(st.positions[-1, 0]) < 1e-12
