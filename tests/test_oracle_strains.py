"""Pins of the oracle's strain measures (orc_rod_strains).

Closed forms and invariants: rest state, uniform stretch, rigid-motion objectivity,
the pure-twist Darboux vector (golden, derived from PAPER.md:238), a constant-Darboux
helix, and second-order convergence to 1/R on a discrete circle.
"""
import json
import os

import numpy as np
import scipy.linalg as sla

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "so3_sign.json")))


def skew_np(v):
    return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])


def straight(N, lhat, Q=np.eye(3)):
    pos = np.arange(N + 1)[:, None] * lhat * Q[2][None, :]
    return np.full(N, lhat), pos, np.tile(Q, (N, 1, 1))


def rand_rot(rng):
    return sla.expm(skew_np(rng.standard_normal(3) * 2))


def test_rest_state(orc):
    rng = np.random.default_rng(0)
    for N in (1, 2, 7):
        lhat, pos, Q = straight(N, 0.25)  # axis-aligned: exact
        e, s, k, f = orc.rod_strains(lhat, pos, Q)
        assert f == 0 and np.array_equal(e, np.ones(N)) and np.array_equal(s, np.zeros((N, 3)))
        assert np.array_equal(k, np.zeros((N - 1, 3)))
        lhat, pos, Q = straight(N, 0.1, rand_rot(rng))  # randomly oriented: round-off only
        e, s, k, f = orc.rod_strains(lhat, pos, Q)
        assert np.max(np.abs(e - 1)) < 1e-13 and np.max(np.abs(s)) < 1e-13
        assert k.size == 0 or np.max(np.abs(k)) < 1e-13


def test_uniform_stretch(orc):
    lhat, pos, Q = straight(5, 0.2)
    e, s, k, _ = orc.rod_strains(lhat, pos * 1.1, Q)
    assert np.allclose(e, 1.1, rtol=0, atol=1e-15)
    assert np.allclose(s, [[0, 0, 0.1]] * 5, rtol=0, atol=1e-15)


def test_objectivity(orc):
    """r -> R r + c, Q -> Q R^T leaves sigma and kappa unchanged (north_star)."""
    rng = np.random.default_rng(1)
    N = 12
    lhat = rng.uniform(0.05, 0.15, N)
    pos = np.cumsum(np.vstack([np.zeros(3), rng.standard_normal((N, 3)) * 0.1]), axis=0)
    Q = np.stack([rand_rot(rng) for _ in range(N)])
    # keep adjacent relative rotations well below pi
    for j in range(1, N):
        Q[j] = sla.expm(skew_np(rng.standard_normal(3) * 0.3)) @ Q[j - 1]
    e0, s0, k0, _ = orc.rod_strains(lhat, pos, Q)
    for _ in range(100):
        R, c = rand_rot(rng), rng.standard_normal(3) * 10
        e1, s1, k1, _ = orc.rod_strains(lhat, pos @ R.T + c, Q @ R.T)
        assert np.max(np.abs(e1 - e0)) < 1e-12
        assert np.max(np.abs(s1 - s0)) < 1e-12 * max(1, np.max(np.abs(s0)))
        assert np.max(np.abs(k1 - k0)) < 1e-12 * max(1, np.max(np.abs(k0)))


def test_pure_twist(orc):
    g = GOLD["pure_twist"]
    tau, N, lhat = g["tau"], 20, 0.05
    s = (np.arange(N) + 0.5) * lhat
    Q = np.stack([np.array([[np.cos(tau * x), np.sin(tau * x), 0], [-np.sin(tau * x), np.cos(tau * x), 0],
                            [0, 0, 1.0]]) for x in s])
    pos = np.arange(N + 1)[:, None] * lhat * np.array([0, 0, 1.0])
    e, sig, k, _ = orc.rod_strains(np.full(N, lhat), pos, Q)
    assert np.allclose(k, np.array(g["kappa"])[None, :], atol=1e-13, rtol=0)
    assert np.allclose(sig, 0, atol=4e-15)


def test_constant_darboux_helix(orc):
    """Q_k = exp(-Dh [kappa]x) Q_{k-1} (built with scipy expm) -> kappa_hat = kappa exactly."""
    rng = np.random.default_rng(2)
    kap = np.array([1.3, -0.4, 2.1])
    N, lhat = 30, 0.03
    Q = [rand_rot(rng)]
    for _ in range(N - 1):
        Q.append(sla.expm(-lhat * skew_np(kap)) @ Q[-1])
    Q = np.stack(Q)
    pos = np.vstack([np.zeros(3), np.cumsum(lhat * Q[:, 2, :], axis=0)])  # edges along d3: sigma = 0
    e, s, k, _ = orc.rod_strains(np.full(N, lhat), pos, Q)
    assert np.allclose(k, kap[None, :], atol=1e-12, rtol=0)
    assert np.max(np.abs(s)) < 1e-14


def circle_rod(R, N):
    """Nodes on a circle of radius R in the x-y plane, element frames with d3 along the chord
    and d1 normal to the plane (tangent-aligned frames)."""
    phi = np.linspace(0, np.pi / 2, N + 1)
    pos = np.stack([R * np.cos(phi), R * np.sin(phi), np.zeros_like(phi)], axis=1)
    chord = pos[1:] - pos[:-1]
    lhat = np.linalg.norm(chord, axis=1)
    t = chord / lhat[:, None]
    d1 = np.tile([0, 0, 1.0], (N, 1))
    d2 = np.cross(t, d1)
    return lhat, pos, np.stack([d1, d2, t], axis=1)


def test_circle_second_order(orc):
    """|kappa_hat| -> 1/R with error O(h^2)."""
    R = 0.7
    errs = []
    for N in (8, 16, 32, 64):
        lhat, pos, Q = circle_rod(R, N)
        e, s, k, _ = orc.rod_strains(lhat, pos, Q)
        errs.append(np.max(np.abs(np.linalg.norm(k, axis=1) - 1.0 / R)))
        assert np.allclose(k[:, 1:], 0, atol=1e-12)        # bending about d1 only
    ratios = np.array(errs[:-1]) / np.array(errs[1:])
    assert np.all(ratios > 3.5), ratios


def test_curvature_matches_continuum_definition(orc):
    """kappa = ax(Q dQ^T/ds) for a smooth frame field Q(s) = expm(s A) Q0,
    differentiated numerically, vs the discrete inverse-Rodrigues curvature."""
    rng = np.random.default_rng(3)
    A = skew_np(np.array([0.8, -1.1, 0.5]))
    Q0 = rand_rot(rng)
    N, lhat = 40, 0.01
    s_el = (np.arange(N) + 0.5) * lhat
    Q = np.stack([(sla.expm(x * A) @ Q0) for x in s_el])
    Qf = lambda x: sla.expm(x * A) @ Q0
    pos = np.vstack([np.zeros(3), np.cumsum(lhat * Q[:, 2, :], axis=0)])
    _, _, k, _ = orc.rod_strains(np.full(N, lhat), pos, Q)
    for kk in (1, N // 2, N - 1):
        x, h = kk * lhat, 1e-6
        dQ = (Qf(x + h) - Qf(x - h)) / (2 * h)
        expect = orc.ax(Qf(x) @ dQ.T)
        assert np.allclose(k[kk - 1], expect, atol=1e-8, rtol=0)
