"""Pins of the muscular-torque traveling wave (reading DESIGN §3 #26):
tau_k(t) = A sin(2 pi (t/T - s_k/lambda) + phi0) at interior nodes, applied as couple pairs.
- net zero: the muscle couples on a rod sum to zero at every instant;
- a static wave (T -> infinity) bends a free rod to the equilibrium curvature kappa_k = tau_k / B
  (couple balance m_k - tau_k = 0 with free ends);
- the wave travels toward +s with phase speed lambda / T.
"""
import dataclasses

import numpy as np

from rodkit import rod


def musc(w, A, T, lam, phi, comp=0):
    R = w.n_rods
    return dataclasses.replace(w, musc_A=np.full(R, A), musc_T=np.full(R, T), musc_lambda=np.full(R, lam),
                               musc_phi=np.full(R, phi), musc_component=comp)


def test_net_zero_and_pattern(orc):
    N, L = 12, 0.6
    w = musc(rod(N=N, L=L), A=2e-3, T=0.5, lam=0.4, phi=0.3, comp=0)
    for t in (0.0, 0.13, 0.41):
        out = orc.rod_loads(w, 0, w.positions, w.velocities, w.directors, w.omega, t)
        C = out["C"]
        assert np.max(np.abs(C.sum(axis=0))) < 1e-18
        s = np.arange(N + 1) * L / N
        tau = 2e-3 * np.sin(2 * np.pi * (t / 0.5 - s / 0.4) + 0.3)
        tau[0] = tau[N] = 0.0                      # only interior nodes carry a muscle torque
        expect = tau[:N] - tau[1:]                 # element j: +tau_j - tau_{j+1}
        assert np.allclose(C[:, 0], expect, rtol=0, atol=1e-17)
        assert np.max(np.abs(C[:, 1:])) < 1e-18


def test_static_wave_equilibrium_curvature(orc):
    N, L, A = 24, 0.3, 2e-5
    w = rod(N=N, L=L, r=0.004, nu=40.0)
    B1 = w.youngs[0] * w.I1[0]
    w = musc(w, A=A, T=1e30, lam=0.2, phi=0.7, comp=0)
    st, s, _, _ = orc.step(w, n_steps=120000, dt=1e-5)
    assert s == 0
    _, _, kap, _ = orc.rod_strains(w.rest_lengths, st.positions, st.directors)
    sk = np.arange(1, N) * L / N
    expect = A * np.sin(0.7 - 2 * np.pi * sk / 0.2) / B1
    assert np.allclose(kap[:, 0], expect, atol=2e-4 * np.max(np.abs(expect))), np.max(np.abs(kap[:, 0] - expect))


def test_wave_travels_forward(orc):
    """Quasi-static response of a soft, strongly damped rod follows the wave: the curvature
    pattern at t + T/4 equals the pattern at t shifted by lambda/4 toward +s."""
    N, L, A, T, lam = 40, 0.4, 1e-5, 4.0, 0.2
    w = rod(N=N, L=L, r=0.004, nu=60.0)
    w = musc(w, A=A, T=T, lam=lam, phi=0.0, comp=0)
    st, s, _, _ = orc.step(w, n_steps=100000, dt=1e-5)
    _, _, k1, _ = orc.rod_strains(w.rest_lengths, st.positions, st.directors)
    st, s, _, _ = orc.step(w, st, n_steps=100000, dt=1e-5)     # + 1 s = T/4
    _, _, k2, _ = orc.rod_strains(w.rest_lengths, st.positions, st.directors)
    shift = int(round((lam / 4) / (L / N)))                     # lambda/4 = 5 elements
    a, b = k1[:-shift, 0], k2[shift:, 0]
    assert np.corrcoef(a, b)[0, 1] > 0.99
