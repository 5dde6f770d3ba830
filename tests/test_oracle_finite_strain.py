"""Pins of the finite-strain and bend-twist terms of Eq. (1b) at e != 1.

Every other dynamics pin runs at e ~ 1 with planar bending (kappa parallel to B kappa), so the
e-powers and the kappa x B kappa term were checked only by reading.  These closed forms fix them:

(a) Constant-Darboux helix with anisotropic bending stiffness (I2 = 3 I1, so kappa x B kappa != 0),
    edges along d3 and stretched.  For a constant curvature the difference term d/ds(B kappa/e^3)
    vanishes and Eq. (1b)'s couple per reference length is kappa x B kappa / e^3.
    - uniform stretch e: interior couple per element = lhat kappa x B kappa / e^3 exactly;
    - alternating stretches e_j in {1.1, 1.3}: the Voronoi dilatation is the mean of the two
      neighbouring edges (eps_k = D_k / Dh_k = 1.2), the same at every
      interior node, so the interior couple is Dh kappa x B kappa / 1.2^3 and the rod-end elements
      carry +-B kappa/1.2^3 (free ends) plus half of it.
(b) Uniformly stretched straight rod (e = 1.25) spinning with two angular-velocity components and a
    uniform local couple c: the element is a rigid body with the incompressible inertia J/e
    ("rho I / e" with I = I_hat / e^2 per current length, DESIGN §3 #5), so Euler's
    body-frame equation (J/e) dw/dt = (J/e) w x w + c gives dw/dt = (J w x w)/J + e c / J.
(c) Uniformly stretching rod (de/dt != 0, e = 1.25) spinning about d3: no couple acts, so the
    angular momentum (J3/e) w3 is conserved (PAPER.md:248 is the (rho I w/e^2) de/dt term of
    d/dt(rho I w / e)), i.e. dw3/dt = w3 (de/dt) / e.
(d) Rest strains: a configuration whose strains equal the given rest strains is load-free
    (PAPER.md:243-247 act on sigma - sigma0 and kappa - kappa0): a stretched and sheared rod with
    sigma0 = its sigma, a stretched helix with kappa0 = its kappa.

Each expected value below comes from these continuum statements, written out with numpy; none
calls the oracle's own arithmetic.  `tools/oracle_mutants.py` shows that plausible mistakes in the
oracle's Eq. (1b) terms fail at least one of these (or an earlier) pin.
"""
import numpy as np
import scipy.linalg as sla

from rodkit import rod


def skew_np(v):
    return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])


def loads(orc, w, pos, vel, Q, om, t=0.0):
    return orc.rod_loads(w, 0, pos, vel, Q, om, t)


def aniso_rod(N, L, r=0.02, E=1e6, G=None):
    w = rod(N=N, L=L, r=r, E=E, G=G)
    w.I2[:] = 3.0 * w.I1                                  # B1 != B2, J1 != J2
    return w


U = 2.0 ** -53


def shear_roundoff(w, lhat, e):
    """Round-off bound of the shear torque lhat (Q t) x S sigma for edges along d3 with sigma =
    (0, 0, e - 1): the transverse components of Q t are O(u), so the couple carries
    ~ lhat S3 |e - 1| u of rounding (a few u; 8 u taken)."""
    return 8 * U * lhat * w.youngs[0] * w.area[0] * max(abs(e - 1.0), 1.0)


def stiffness(w):
    E, G, I1, I2 = w.youngs[0], w.shear_mod[0], w.I1[0], w.I2[0]
    return np.array([E * I1, E * I2, G * (I1 + I2)])


def inertia(w, lhat):
    rho, I1, I2 = w.density[0], w.I1[0], w.I2[0]
    return rho * lhat * np.array([I1, I2, I1 + I2])


def helix(kap, N, lhat, stretches, Q0):
    """Frames Q_k = expm(-lhat [kappa]x) Q_{k-1} (constant Darboux vector kappa per reference length,
    the rotation sign of PAPER.md:238-239 / DESIGN §3 #2); edge j = stretches[j] * lhat * d3_j."""
    Q = [Q0]
    for _ in range(N - 1):
        Q.append(sla.expm(-lhat * skew_np(kap)) @ Q[-1])
    Q = np.stack(Q)
    edges = (np.asarray(stretches)[:, None] * lhat) * Q[:, 2, :]
    pos = np.vstack([np.zeros(3), np.cumsum(edges, axis=0)])
    return pos, Q


KAP = np.array([1.3, -0.4, 2.1])


def test_helix_uniform_stretch_couple(orc):
    """(a) e = 1.25 everywhere: interior C_j = lhat kappa x B kappa / e^3."""
    N, L, e = 12, 0.6, 1.25
    lhat = L / N
    w = aniso_rod(N, L)
    B = stiffness(w)
    Q0 = sla.expm(skew_np([0.3, -0.8, 0.5]))
    pos, Q = helix(KAP, N, lhat, np.full(N, e), Q0)
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    expect = lhat * np.cross(KAP, B * KAP) / e ** 3
    scale = np.max(np.abs(B * KAP))
    assert np.max(np.abs(expect)) > 1e-3 * scale           # the bend-twist coupling is really there
    assert np.max(np.abs(out["C"][1:-1] - expect[None, :])) <= 1e-12 * scale + shear_roundoff(w, lhat, e)


def test_helix_alternating_stretch_couple(orc):
    """(a) e_j alternating 1.1 / 1.3: Voronoi dilatation 1.2 from the neighbouring lengths; interior
    C_j = Dh kappa x B kappa / 1.2^3, end elements +-B kappa / 1.2^3 + (1/2) Dh kappa x B kappa / 1.2^3,
    and alpha_j = e_j C_j / J_j (the rho I / e on the left of Eq. (1b))."""
    N, L = 12, 0.6
    lhat = L / N
    w = aniso_rod(N, L)
    B = stiffness(w)
    J = inertia(w, lhat)
    ej = np.where(np.arange(N) % 2 == 0, 1.1, 1.3)
    Q0 = sla.expm(skew_np([-1.1, 0.2, 0.7]))
    pos, Q = helix(KAP, N, lhat, ej, Q0)
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    eps = 1.2
    m = B * KAP / eps ** 3                                   # bending moment, every interior node
    beta = lhat * np.cross(KAP, m)
    tol = 1e-12 * np.max(np.abs(m)) + shear_roundoff(w, lhat, 1.3)
    C = out["C"]
    assert np.max(np.abs(C[1:-1] - beta[None, :])) <= tol
    assert np.max(np.abs(C[0] - (m + 0.5 * beta))) <= tol
    assert np.max(np.abs(C[-1] - (-m + 0.5 * beta))) <= tol
    # angular acceleration: (J/e) dw/dt = C  (w = 0, no damping)
    expect_alpha = ej[:, None] * C / J[None, :]
    assert np.allclose(out["alpha"], expect_alpha, rtol=1e-13, atol=0)
    # and the dilatation entering alpha is the element's own e_j, not the Voronoi mean
    assert np.max(np.abs(out["alpha"][1:-1] - ej[1:-1, None] * beta[None, :] / J[None, :])) \
        <= 1.3 * tol / np.min(J)


def test_stretched_rigid_body_euler(orc):
    """(b) e = 1.25, w = (w1, w2, 0) uniform, uniform local couple c: dw/dt = (J w x w)/J + e c/J."""
    N, L, e = 4, 0.4, 1.25
    lhat = L / N
    Q0 = sla.expm(skew_np([0.9, 0.1, -0.6]))
    w = aniso_rod(N, L)
    J = inertia(w, lhat)
    pos, Q = helix(np.zeros(3), N, lhat, np.full(N, e), Q0)
    om = np.tile([0.4, -0.7, 0.0], (N, 1))
    c = np.array([2e-7, -1e-7, 3e-7])
    w.ext_couple = np.tile(c, (N, 1))
    out = loads(orc, w, pos, np.zeros_like(pos), Q, om)
    euler = np.cross(J * om[0], om[0]) / J
    assert abs(euler[2]) > 0.1                              # the gyroscopic term is really there
    expect = euler + e * c / J
    tol = 1e-13 * np.max(np.abs(expect)) + e * shear_roundoff(w, lhat, e) / np.min(J)
    assert tol < 1e-5 * np.min(np.abs(expect))
    assert np.max(np.abs(out["alpha"] - expect[None, :])) <= tol


def test_stretching_spin_conserves_angular_momentum(orc):
    """(c) e = 1.25 and de/dt = 0.8 s^-1 on every element, w = w3 d3: dw3/dt = w3 (de/dt) / e."""
    N, L, e, edot, w3 = 3, 0.3, 1.25, 0.8, 2.0
    lhat = L / N
    Q0 = sla.expm(skew_np([0.2, 0.5, -0.3]))
    w = aniso_rod(N, L)
    pos, Q = helix(np.zeros(3), N, lhat, np.full(N, e), Q0)
    d3 = Q0[2]
    vel = (edot * lhat * np.arange(N + 1))[:, None] * d3[None, :]  # t.(v_{j+1}-v_j)/lhat = edot
    om = np.tile([0.0, 0.0, w3], (N, 1))
    out = loads(orc, w, pos, vel, Q, om)
    tol = 1e-13 * w3 * edot + e * shear_roundoff(w, lhat, e) / np.min(inertia(w, lhat))
    assert tol < 1e-5 * w3 * edot
    assert np.max(np.abs(out["alpha"][:, 2] - w3 * edot / e)) <= tol
    assert np.max(np.abs(out["alpha"][:, :2])) <= tol


def test_rest_shear_stretch_is_load_free(orc):
    """(d) A straight rod stretched by e = 1.2 and sheared (edges tilted against d3) carries no load
    when sigma0 equals its strain sigma = e Q t - e3."""
    N, L = 6, 0.6
    lhat = L / N
    w = aniso_rod(N, L)
    Q0 = sla.expm(skew_np([0.4, -0.2, 0.9]))
    tilt = np.array([0.05, -0.03, 1.0])
    tilt /= np.linalg.norm(tilt)                            # local edge direction
    e = 1.2
    edge = e * lhat * (Q0.T @ tilt)                          # lab edge vector
    pos = np.arange(N + 1)[:, None] * edge[None, :]
    Q = np.tile(Q0, (N, 1, 1))
    sigma = e * tilt - np.array([0, 0, 1.0])
    w.rest_sigma = np.tile(sigma, (N, 1))
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    S3 = w.youngs[0] * w.area[0]
    assert np.max(np.abs(out["F"])) <= 1e-12 * S3
    assert np.max(np.abs(out["C"])) <= 1e-12 * S3 * lhat
    # without the rest strain the same state is loaded (the check above is not vacuous)
    w.rest_sigma = None
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    assert np.max(np.abs(out["F"])) > 1e-3 * S3


def test_rest_curvature_helix_is_load_free(orc):
    """(d) The stretched helix of (a) with kappa0 = kappa and sigma0 = (0, 0, e - 1) is load-free."""
    N, L, e = 10, 0.5, 1.15
    lhat = L / N
    w = aniso_rod(N, L)
    pos, Q = helix(KAP, N, lhat, np.full(N, e), sla.expm(skew_np([0.1, 0.2, 0.3])))
    w.rest_kappa = np.tile(KAP, (N - 1, 1))
    w.rest_sigma = np.tile([0.0, 0.0, e - 1.0], (N, 1))
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    B = stiffness(w)
    assert np.max(np.abs(out["C"])) <= 1e-11 * np.max(B * np.abs(KAP))
    assert np.max(np.abs(out["F"])) <= 1e-11 * w.youngs[0] * w.area[0]


def test_nonuniform_lhat_helix(orc):
    """A smooth frame field of constant Darboux vector kappa sampled at the element centres of a rod
    with non-uniform rest lengths: the centres of elements k-1 and k are (lhat_{k-1} + lhat_k)/2
    apart (the Voronoi length Dh_k), so kappa_hat = kappa exactly, the moment B kappa is uniform and
    the interior couples are the averaged bend-twist terms (1/2)(Dh_j + Dh_{j+1}) kappa x B kappa."""
    N = 9
    lh = np.array([0.03, 0.05, 0.02, 0.07, 0.04, 0.03, 0.06, 0.025, 0.045])
    w = aniso_rod(N, lh.sum())
    w.rest_lengths = lh.copy()
    B = stiffness(w)
    centres = np.cumsum(lh) - 0.5 * lh
    Q0 = sla.expm(skew_np([0.5, 0.1, -0.9]))
    Q = np.stack([sla.expm(-s * skew_np(KAP)) @ Q0 for s in centres])
    pos = np.vstack([np.zeros(3), np.cumsum(lh[:, None] * Q[:, 2, :], axis=0)])
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    Dh = 0.5 * (lh[:-1] + lh[1:])                      # Voronoi k = 1..N-1
    kxBk = np.cross(KAP, B * KAP)
    tol = 1e-11 * np.max(np.abs(B * KAP))
    for j in range(1, N - 1):
        expect = 0.5 * (Dh[j - 1] + Dh[j]) * kxBk
        assert np.max(np.abs(out["C"][j] - expect)) <= tol, j
    assert np.max(np.abs(out["C"][0] - (B * KAP + 0.5 * Dh[0] * kxBk))) <= tol
    assert np.max(np.abs(out["C"][-1] - (-B * KAP + 0.5 * Dh[-1] * kxBk))) <= tol


def test_composite_rod_uniform_moment(orc):
    """A rod whose elements alternate between two bending stiffnesses, bent about d1 by the exact
    piecewise-constant curvature M / B1(s) of a uniform moment M (the relative rotation of two
    element centres is M (lhat_{k-1}/(2 B_{k-1}) + lhat_k/(2 B_k))): every Voronoi node carries
    m = M, so interior couples vanish and the free ends carry +-M (DESIGN §3 #9)."""
    N, lhat, M = 8, 0.05, 2e-3
    r = 0.02
    E = np.where(np.arange(N) % 2 == 0, 1e6, 4e6)
    A, I1 = np.pi * r * r, np.pi * r ** 4 / 4
    w = rod(N=N, L=N * lhat, r=r)
    w.density = np.full(N, 1000.0)
    w.area, w.I1, w.I2 = np.full(N, A), np.full(N, I1), np.full(N, 3 * I1)
    w.youngs, w.shear_mod, w.alpha_c = E.copy(), E / 3.0, np.full(N, 4.0 / 3.0)
    B1 = E * I1
    Q = [sla.expm(skew_np([0.2, -0.4, 0.3]))]
    for k in range(1, N):
        dth = M * (lhat / (2 * B1[k - 1]) + lhat / (2 * B1[k]))
        Q.append(sla.expm(-dth * skew_np([1.0, 0, 0])) @ Q[-1])
    Q = np.stack(Q)
    pos = np.vstack([np.zeros(3), np.cumsum(lhat * Q[:, 2, :], axis=0)])
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    tol = 1e-11 * M + 8 * U * np.max(E) * A * lhat        # + shear-torque round-off
    assert np.max(np.abs(out["C"][1:-1])) <= tol
    assert np.max(np.abs(out["C"][0] - [M, 0, 0])) <= tol
    assert np.max(np.abs(out["C"][-1] - [-M, 0, 0])) <= tol


def test_timoshenko_shear_force(orc):
    """A uniformly sheared straight rod (edges at angle gamma to d3 in the d1-d3 plane, no stretch
    of the centreline): the end node carries the Timoshenko shear force alpha_c G A sin(gamma) along
    d1 and the axial force E A (cos(gamma) - 1) along d3 (S = diag(alpha_c G A, alpha_c G A, E A),
    PAPER.md:239; n = Q^T S sigma / e with e = 1)."""
    N, L, gamma = 5, 0.5, 0.01
    w = rod(N=N, L=L, r=0.02)
    lhat = L / N
    Q0 = sla.expm(skew_np([0.3, 0.6, -0.2]))
    tl = np.array([np.sin(gamma), 0.0, np.cos(gamma)])    # local edge direction
    pos = np.arange(N + 1)[:, None] * (lhat * (Q0.T @ tl))[None, :]
    Q = np.tile(Q0, (N, 1, 1))
    out = loads(orc, w, pos, np.zeros_like(pos), Q, np.zeros((N, 3)))
    GA = w.shear_mod[0] * w.area[0]
    EA = w.youngs[0] * w.area[0]
    n_local = np.array([w.alpha_c[0] * GA * np.sin(gamma), 0.0, EA * (np.cos(gamma) - 1.0)])
    expect = Q0.T @ n_local                                # F_0 = n_0 (lab)
    assert np.max(np.abs(out["F"][0] - expect)) <= 1e-10 * np.max(np.abs(n_local))
    assert np.max(np.abs(out["F"][-1] + expect)) <= 1e-10 * np.max(np.abs(n_local))
