"""Pins of the oracle's contact model (
readings DESIGN §3 #27): exact segment distance, exhaustive detection with same-rod exclusion,
penalty normal force, regularised Coulomb friction, half-space boundary."""
import dataclasses

import numpy as np
import pytest
from scipy.optimize import minimize

import workloads as W
from rodkit import concat, rod


def brute_min(p0, p1, q0, q1):
    f = lambda x: np.sum((p0 + x[0] * (p1 - p0) - q0 - x[1] * (q1 - q0)) ** 2)
    best = min((minimize(f, x0, bounds=[(0, 1), (0, 1)], method="L-BFGS-B", options={"ftol": 1e-16, "gtol": 1e-14})
                for x0 in ([0.5, 0.5], [0, 0], [1, 1], [0, 1], [1, 0])), key=lambda r: r.fun)
    return np.sqrt(max(best.fun, 0.0))


def test_segment_closest_special_cases(orc):
    s, t, d = orc.segment_closest([0, 0, 0], [1, 0, 0], [0, 0.3, 0], [1, 0.3, 0])   # parallel, offset 0.3
    assert d == pytest.approx(0.3, abs=1e-15)
    s, t, d = orc.segment_closest([-1, 0, 0], [1, 0, 0], [0, -1, 0], [0, 1, 0])     # crossing
    assert d == 0.0 and s == 0.5 and t == 0.5
    s, t, d = orc.segment_closest([0, 0, 0], [0, 0, 0], [1, 1, 0], [1, 1, 0])       # two points
    assert d == pytest.approx(np.sqrt(2), abs=1e-15)


def test_segment_closest_vs_independent_minimiser(orc):
    rng = np.random.default_rng(0)
    for _ in range(300):
        p0, p1, q0, q1 = rng.standard_normal((4, 3))
        s, t, d = orc.segment_closest(p0, p1, q0, q1)
        assert 0 <= s <= 1 and 0 <= t <= 1
        x = p0 + s * (p1 - p0) - q0 - t * (q1 - q0)
        assert np.linalg.norm(x) == pytest.approx(d, abs=1e-14)
        assert d <= brute_min(p0, p1, q0, q1) + 1e-9
        s2, t2, d2 = orc.segment_closest(q0, q1, p0, p1)                              # swap symmetry
        assert d2 == pytest.approx(d, abs=1e-14)


def two_rods(gap, angle=np.pi / 2, N=8, L=0.4, r=0.01, **kw):
    """Rod A along x at z = 0; rod B along direction (cos a, sin a, 0) at height z = 2r + gap.
    The rods cross at the origin, which is the middle of element N/2 of each rod (so exactly
    one element pair is in contact)."""
    lh = L / N
    A = rod(N=N, L=L, r=r, Q=np.array([[0, 0, -1.0], [0, 1.0, 0], [1.0, 0, 0]]),
            base=(-L / 2 - lh / 2, 0, 0), **kw)
    d = np.array([np.cos(angle), np.sin(angle), 0.0])
    d1 = np.array([0, 0, 1.0])
    Qb = np.stack([d1, np.cross(d, d1), d])
    B = rod(N=N, L=L, r=r, Q=Qb, base=tuple(-(L / 2 + lh / 2) * d + np.array([0, 0, 2 * r + gap])), **kw)
    return concat([A, B])


def test_detection_and_exclusion(orc):
    w = two_rods(-1e-4)
    w.contact = W.Contact(k_n=1e3)
    pairs, gaps = orc.contact_pairs(w, w.positions)
    assert pairs.tolist() == [[4, 12]]                                 # element 4 of A, element 4 of B
    assert np.min(gaps) == pytest.approx(-1e-4, abs=1e-12)
    w2 = two_rods(+1e-4)
    w2.contact = W.Contact(k_n=1e3)
    assert len(orc.contact_pairs(w2, w2.positions)[0]) == 0
    # a straight slender rod never touches itself: elements within the exclusion stencil are
    # skipped, farther ones are > 2 lhat apart (radius < lhat / 2 here)
    w3 = rod(N=20, L=0.2, r=0.004)
    w3.contact = W.Contact(k_n=1e3)
    assert len(orc.contact_pairs(w3, w3.positions)[0]) == 0


def test_static_penetration_force_and_third_law(orc):
    delta, k = 2e-4, 5e3
    w = two_rods(-delta)
    w.contact = W.Contact(k_n=k, gamma_n=10.0, mu_s=0.5, mu_k=0.4)
    F = orc.contact_forces(w, w.positions, w.velocities)
    assert np.allclose(F.sum(axis=0), 0.0, atol=1e-15)
    fa, fb = F[:9].sum(axis=0), F[9:].sum(axis=0)
    assert np.allclose(fb, [0, 0, k * delta], rtol=1e-10, atol=1e-15)   # B pushed up, |F| = k delta
    assert np.allclose(fa, -fb, rtol=0, atol=1e-15)


def test_rest_on_floor_reaction_equals_weight(orc):
    """A horizontal rod settles on the half-space z >= 0 under gravity: plane reaction = weight
    (SPEC.md:412)."""
    N, L, r = 10, 0.2, 0.005
    w = rod(N=N, L=L, r=r, Q=np.array([[0, 0, -1.0], [0, 1.0, 0], [1.0, 0, 0]]), base=(0, 0, r), nu=30.0,
            g=(0, 0, -9.81))
    w.contact = W.Contact(k_n=2e3, gamma_n=0.5, plane_n=np.array([0, 0, 1.0]), plane_d=0.0)
    st, s, _, _ = orc.step(w, n_steps=40000, dt=1e-5)
    assert s == 0
    F = orc.contact_forces(w, st.positions, st.velocities)
    weight = w.density[0] * w.area[0] * L * 9.81
    assert F[:, 2].sum() == pytest.approx(weight, rel=1e-2)
    assert np.max(np.abs(st.velocities)) < 1e-4


def test_coulomb_sliding_deceleration(orc):
    """A rod sliding along the floor decelerates at mu_k g (kinetic branch)."""
    N, L, r, mu, v0 = 10, 0.2, 0.005, 0.3, 0.1
    w = rod(N=N, L=L, r=r, Q=np.array([[0, 0, -1.0], [0, 1.0, 0], [1.0, 0, 0]]), base=(0, 0, r), nu=0.0,
            g=(0, 0, -9.81))
    w.contact = W.Contact(k_n=2e3, gamma_n=0.5, mu_s=mu, mu_k=mu, v_stick=1e-4, plane_n=np.array([0, 0, 1.0]))
    w.velocities[:, 0] = v0
    st, s, _, _ = orc.step(w, n_steps=2000, dt=1e-5)                  # settle the contact (0.02 s)
    v1 = st.velocities[:, 0].mean()
    t1 = st.t
    st, s, _, _ = orc.step(w, st, n_steps=1000, dt=1e-5)
    v2 = st.velocities[:, 0].mean()
    decel = (v1 - v2) / (st.t - t1)
    assert decel == pytest.approx(mu * 9.81, rel=1e-2)


def test_head_on_impact_conserves_momentum(orc):
    w = two_rods(5e-4, angle=np.pi / 3)
    w.contact = W.Contact(k_n=5e3, gamma_n=2.0, mu_s=0.3, mu_k=0.2)
    nB = slice(9, 18)
    w.velocities[nB, 2] = -0.5                                          # B falls onto A
    P0 = orc.energy(w)[6:9]
    st, s, _, _ = orc.step(w, n_steps=3000, dt=1e-6)
    assert s == 0
    pairs, _ = orc.contact_pairs(w, st.positions)
    P1 = orc.energy(w, st)[6:9]
    assert np.allclose(P1, P0, rtol=0, atol=1e-12 * np.abs(P0).max())
    assert st.velocities[nB, 2].mean() > -0.5                          # B was slowed by the contact


def test_fibres_recipe(orc):
    """The NEXT-4 contact workload: neighbouring layers of a stack overlap by overlap +- overlap/4
    at every crossing, the bottom layer presses into the floor, and two neighbouring stacks never
    touch (so a stack is an independent sub-problem, used for full-size parity and sharding)."""
    c = W.FIBRES
    per = c["layers"] * c["per_layer"]
    w = W.make("fibres", n_rods=2 * per)
    pairs, gaps = orc.contact_pairs(w, w.positions)
    assert len(pairs) > 0
    assert np.all(gaps < -c["overlap"] / 4) and np.all(gaps > -7 * c["overlap"] / 4)
    rod_of = np.repeat(np.arange(w.n_rods), w.n_elems)
    assert np.all(rod_of[pairs[:, 0]] // per == rod_of[pairs[:, 1]] // per)      # no pair across stacks
    # each crossing of neighbouring layers in stack 0 is one contact (16 x 16 crossings x 15 layer pairs,
    # a crossing at an element boundary can count twice)
    st0 = pairs[rod_of[pairs[:, 0]] < per]
    assert 16 * 16 * 15 <= len(st0) <= 2 * 16 * 16 * 15
    z0 = w.positions[:, 2][np.repeat(np.arange(w.n_rods), w.n_elems + 1) % per < c["per_layer"]]
    assert np.all(z0 < c["radius"]) and np.all(z0 > c["radius"] - c["overlap"])
