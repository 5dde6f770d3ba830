"""Seeded synthetic workloads (cfg1..cfg5) shared by the oracle and the CUDA path.

This module holds *no* arithmetic of the rod method (no Rodrigues map, no
strains, no forces): it only draws random numbers and lays out initial rods
(straight centrelines, director frames from unit quaternions, circular
cross-sections).  Both `oracle/` and the product path consume its arrays
verbatim, which is the only thing the two sides share.

Recipe: SURVEY.md §8 D.1 (configs from BASELINE.json `configs[0..4]`).
- RNG: numpy Generator(Philox(260513766 + k)) for cfg k (k = 1..5).
- Draw order: per-rod scalars, per-rod frames, per-element perturbations,
  per-node velocities.
- "Uniform SO(3)": a normalised N(0,1)^4 quaternion turned into a matrix whose
  rows are the directors d1, d2, d3.
- Straight rod along unit d: r_i = r0 + (sum_{j<i} lhat_j) d, every Q_j has d3 = d.
- Circular section of radius r: A = pi r^2, I1 = I2 = pi r^4 / 4
  ("I = diag{I1, I2, I1+I2}").

Array conventions (the canonical, C-ABI order; see include/er.h):
- positions / velocities: [n_nodes, 3] lab frame, nodes of rod r are contiguous
  and rod r owns n_elems[r] + 1 nodes;
- directors: [n_elems, 3, 3], row a = d_{a+1} in lab coordinates;
- omega: [n_elems, 3] local frame;
- rest_kappa: [n_voronoi, 3] local frame (rod r owns n_elems[r] - 1 entries);
- per-rod material arrays: [n_rods].
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

SEED_BASE = 260513766
CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


@dataclasses.dataclass
class Contact:
    """Contact parameters (NEXT-4; reading DESIGN §3 #27): penalty k_n (<= 0: min(E_A r_A, E_B r_B)),
    normal damping gamma_n, regularised Coulomb friction (mu_s, mu_k, v_stick), contact radius per
    rod (None = sqrt(A/pi)), same-rod exclusion |j - k| <= exclude, optional half-space n.x >= d."""
    k_n: float = 0.0
    gamma_n: float = 0.0
    mu_s: float = 0.0
    mu_k: float = 0.0
    v_stick: float = 1e-4
    radius: Optional[np.ndarray] = None
    exclude: int = 2
    plane_n: Optional[np.ndarray] = None
    plane_d: float = 0.0


@dataclasses.dataclass
class Workload:
    name: str
    n_elems: np.ndarray            # int32 [R]
    rest_lengths: np.ndarray       # f64 [E]
    density: np.ndarray            # f64 [R] volumetric (kg/m^3), SURVEY C.4 #6
    area: np.ndarray               # f64 [R]
    I1: np.ndarray                 # f64 [R]
    I2: np.ndarray                 # f64 [R]
    youngs: np.ndarray             # f64 [R]
    shear_mod: np.ndarray          # f64 [R]
    alpha_c: np.ndarray            # f64 [R]
    positions: np.ndarray          # f64 [Nn, 3]
    velocities: np.ndarray         # f64 [Nn, 3]
    directors: np.ndarray          # f64 [E, 3, 3]
    omega: np.ndarray              # f64 [E, 3]
    clamp: np.ndarray              # int8 [R]: -1 free, 0 clamp s=0 end, 1 clamp s=L end
    gravity: np.ndarray            # f64 [3]
    damping: np.ndarray            # f64 [R] (s^-1, rate form)
    tip_force: Optional[np.ndarray] = None    # f64 [R, 3] lab, constant
    rest_sigma: Optional[np.ndarray] = None   # f64 [E, 3]
    rest_kappa: Optional[np.ndarray] = None   # f64 [V, 3] static part
    act_A: Optional[np.ndarray] = None        # f64 [R]
    act_f: Optional[np.ndarray] = None        # f64 [R]
    act_L: Optional[np.ndarray] = None        # f64 [R]
    act_component: int = 0
    dt: float = 1e-5
    n_steps: int = 1
    t0: float = 0.0
    # magnetic couple (NEXT-2): per-element m̄ (local) and field b(t)
    magnetization: Optional[np.ndarray] = None  # f64 [E, 3]
    b_field: Optional[np.ndarray] = None        # f64 [3] amplitude (lab)
    b_omega: float = 0.0                        # rad/s, b(t) = R_axis(b_omega t) b_field
    b_axis: Optional[np.ndarray] = None         # f64 [3] rotation axis of b(t); None = lab z
    # muscular torque wave (NEXT-3): tau = A sin(2 pi (t/T - s/lambda) + phi)
    musc_A: Optional[np.ndarray] = None         # f64 [R]
    musc_T: Optional[np.ndarray] = None         # f64 [R]
    musc_lambda: Optional[np.ndarray] = None    # f64 [R]
    musc_phi: Optional[np.ndarray] = None       # f64 [R]
    musc_component: int = 0
    contact: Optional[Contact] = None           # NEXT-4: rods interact through contact
    ext_force: Optional[np.ndarray] = None      # [n_nodes, 3] lab, N: f of Eq. (1a) per node
    ext_couple: Optional[np.ndarray] = None     # [n_elems, 3] local, N m: c-bar of Eq. (1b) per element

    # ---- layout helpers (integer bookkeeping only) ----
    @property
    def n_rods(self) -> int:
        return int(self.n_elems.shape[0])

    @property
    def n_elems_total(self) -> int:
        return int(self.n_elems.sum())

    @property
    def n_nodes_total(self) -> int:
        return self.n_elems_total + self.n_rods

    @property
    def n_voronoi_total(self) -> int:
        return self.n_elems_total - self.n_rods

    def elem_offsets(self) -> np.ndarray:
        o = np.zeros(self.n_rods + 1, dtype=np.int64)
        np.cumsum(self.n_elems, out=o[1:])
        return o

    def node_offsets(self) -> np.ndarray:
        return self.elem_offsets() + np.arange(self.n_rods + 1, dtype=np.int64)

    def voronoi_offsets(self) -> np.ndarray:
        return self.elem_offsets() - np.arange(self.n_rods + 1, dtype=np.int64)

    def element_steps(self, n_steps: Optional[int] = None) -> int:
        return self.n_elems_total * (self.n_steps if n_steps is None else n_steps)

    def subset(self, rods) -> "Workload":
        """Rods are independent (no contact): any subset is a valid workload."""
        rods = np.asarray(rods, dtype=np.int64)
        eo, no, vo = self.elem_offsets(), self.node_offsets(), self.voronoi_offsets()

        def gather(off, arr):
            if arr is None:
                return None
            idx = np.concatenate([np.arange(off[r], off[r + 1]) for r in rods]) if len(rods) else np.zeros(0, np.int64)
            return np.ascontiguousarray(arr[idx])

        def per_rod(arr):
            return None if arr is None else np.ascontiguousarray(arr[rods])

        return dataclasses.replace(
            self,
            name=f"{self.name}[subset:{len(rods)}]",
            n_elems=per_rod(self.n_elems),
            rest_lengths=gather(eo, self.rest_lengths),
            density=per_rod(self.density), area=per_rod(self.area),
            I1=per_rod(self.I1), I2=per_rod(self.I2), youngs=per_rod(self.youngs),
            shear_mod=per_rod(self.shear_mod), alpha_c=per_rod(self.alpha_c),
            positions=gather(no, self.positions), velocities=gather(no, self.velocities),
            directors=gather(eo, self.directors), omega=gather(eo, self.omega),
            clamp=per_rod(self.clamp), damping=per_rod(self.damping),
            tip_force=per_rod(self.tip_force),
            rest_sigma=gather(eo, self.rest_sigma), rest_kappa=gather(vo, self.rest_kappa),
            act_A=per_rod(self.act_A), act_f=per_rod(self.act_f), act_L=per_rod(self.act_L),
            magnetization=gather(eo, self.magnetization),
            ext_force=gather(no, self.ext_force), ext_couple=gather(eo, self.ext_couple),
            musc_A=per_rod(self.musc_A), musc_T=per_rod(self.musc_T),
            musc_lambda=per_rod(self.musc_lambda), musc_phi=per_rod(self.musc_phi),
            contact=None if self.contact is None else dataclasses.replace(
                self.contact, radius=per_rod(self.contact.radius)),
        )

    def copy_state(self):
        return (self.positions.copy(), self.velocities.copy(),
                self.directors.copy(), self.omega.copy())


# ---------------------------------------------------------------------------
# frame construction helpers (input layout only; not the method's rotation map)
# ---------------------------------------------------------------------------

def quat_to_rows(q: np.ndarray) -> np.ndarray:
    """Unit quaternions [..., 4] (w, x, y, z) -> proper orthogonal matrices [..., 3, 3].

    The textbook quaternion-to-matrix formula; the rows are used as d1, d2, d3."""
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    M = np.empty(q.shape[:-1] + (3, 3))
    M[..., 0, 0] = 1 - 2 * (y * y + z * z)
    M[..., 0, 1] = 2 * (x * y - z * w)
    M[..., 0, 2] = 2 * (x * z + y * w)
    M[..., 1, 0] = 2 * (x * y + z * w)
    M[..., 1, 1] = 1 - 2 * (x * x + z * z)
    M[..., 1, 2] = 2 * (y * z - x * w)
    M[..., 2, 0] = 2 * (x * z - y * w)
    M[..., 2, 1] = 2 * (y * z + x * w)
    M[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return M


def uniform_so3(rng: np.random.Generator, n: int) -> np.ndarray:
    return quat_to_rows(rng.standard_normal((n, 4)))


def axis_angle_quat(axis: np.ndarray, angle: np.ndarray) -> np.ndarray:
    axis = axis / np.linalg.norm(axis, axis=-1, keepdims=True)
    h = 0.5 * angle
    return np.concatenate([np.cos(h)[..., None], np.sin(h)[..., None] * axis], axis=-1)


def complete_frame(t: np.ndarray) -> np.ndarray:
    """Unit tangents [n,3] -> frames [n,3,3] with rows d1, d2, d3 = t."""
    a = np.zeros_like(t)
    use_e2 = np.abs(t[:, 0]) > 0.9
    a[~use_e2, 0] = 1.0
    a[use_e2, 1] = 1.0
    d1 = np.cross(a, t)
    d1 /= np.linalg.norm(d1, axis=1, keepdims=True)
    d2 = np.cross(t, d1)
    return np.stack([d1, d2, t], axis=1)


def circular_section(radius: np.ndarray):
    area = math.pi * radius ** 2
    inertia = math.pi * radius ** 4 / 4.0
    return area, inertia, inertia.copy()


def straight_rods(n_elems: np.ndarray, lhat_per_rod: np.ndarray, base: np.ndarray,
                  d3: np.ndarray) -> np.ndarray:
    """Node positions of straight rods: r_i = base + i*lhat*d3 (uniform rest length)."""
    R = n_elems.shape[0]
    nn = n_elems.astype(np.int64) + 1
    rod_of_node = np.repeat(np.arange(R), nn)
    starts = np.zeros(R, np.int64)
    np.cumsum(nn[:-1], out=starts[1:])
    i = np.arange(int(nn.sum()), dtype=np.int64) - starts[rod_of_node]
    return base[rod_of_node] + (i * lhat_per_rod[rod_of_node])[:, None] * d3[rod_of_node]


def _expand(per_rod: np.ndarray, n_elems: np.ndarray) -> np.ndarray:
    return np.repeat(per_rod, n_elems.astype(np.int64), axis=0)


def _rod_material(R, radius, E, rho=1000.0, alpha_c=4.0 / 3.0):
    radius = np.broadcast_to(np.asarray(radius, float), (R,)).copy()
    E = np.broadcast_to(np.asarray(E, float), (R,)).copy()
    area, I1, I2 = circular_section(radius)
    return dict(density=np.full(R, rho), area=area, I1=I1, I2=I2, youngs=E,
                shear_mod=E / 3.0, alpha_c=np.full(R, alpha_c))


# ---------------------------------------------------------------------------
# the five configs (BASELINE.json configs[0..4])
# ---------------------------------------------------------------------------

EXTRA_CONFIGS = ("cilia8", "ciliafarm", "fibres")


def make(name: str, n_rods: Optional[int] = None, n_steps: Optional[int] = None) -> Workload:
    """Build config `name` ("cfg1".."cfg5", or the NEXT-2 cilia workloads).  `n_rods` shrinks
    the batch (a different seeded draw of the same recipe); use `.subset()` to sample rods of the
    full draw."""
    if name in EXTRA_CONFIGS:
        w = _fibres(n_rods) if name == "fibres" else _cilia(name, n_rods)
        if n_steps is not None:
            w.n_steps = int(n_steps)
        return w
    k = CONFIG_NAMES.index(name) + 1
    rng = np.random.Generator(np.random.Philox(SEED_BASE + k))
    fn = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5}[k]
    w = fn(rng, n_rods)
    if n_steps is not None:
        w.n_steps = int(n_steps)
    return w


def _cfg1(rng, n_rods):
    # Single cantilever: L=1, r=0.01, rho=1000, E=1e6, G=E/3, straight +z, Q=I,
    # clamp s=0, tip force 1e-3 N along +x, damping 0.1, dt=1e-4, 20000 steps.
    R = 1 if n_rods is None else int(n_rods)
    N = 100
    n_elems = np.full(R, N, np.int32)
    lhat = np.full(R, 1.0 / N)
    mat = _rod_material(R, 0.01, 1e6)
    d3 = np.tile(np.array([0.0, 0.0, 1.0]), (R, 1))
    base = np.zeros((R, 3))
    base[:, 0] = np.arange(R) * 0.1
    pos = straight_rods(n_elems, lhat, base, d3)
    dirs = np.tile(np.eye(3), (R * N, 1, 1))
    tip = np.tile(np.array([1e-3, 0.0, 0.0]), (R, 1))
    return Workload("cfg1", n_elems, _expand(lhat, n_elems), **mat,
                    positions=pos, velocities=np.zeros_like(pos), directors=dirs,
                    omega=np.zeros((R * N, 3)), clamp=np.zeros(R, np.int8),
                    gravity=np.zeros(3), damping=np.full(R, 0.1), tip_force=tip,
                    dt=1e-4, n_steps=20000)


def _cfg2(rng, n_rods):
    # 4096 free rods x 50 elements, L=1, r=0.01, E log-uniform [1e5,1e7],
    # random unit tangents, directors perturbed by rotations of angle <= 0.05,
    # node velocities N(0, 1e-3), gravity -9.81 z, damping 0.05, dt=1e-5, 10000 steps.
    R = 4096 if n_rods is None else int(n_rods)
    N = 50
    n_elems = np.full(R, N, np.int32)
    lhat = np.full(R, 1.0 / N)
    E = 10.0 ** rng.uniform(5.0, 7.0, R)                      # per-rod scalars
    mat = _rod_material(R, 0.01, E)
    t = rng.standard_normal((R, 3))                           # per-rod frames
    t /= np.linalg.norm(t, axis=1, keepdims=True)
    Qb = complete_frame(t)
    axis = rng.standard_normal((R * N, 3))                    # per-element perturbations
    ang = rng.uniform(0.0, 0.05, R * N)
    P = quat_to_rows(axis_angle_quat(axis, ang))
    dirs = np.einsum("eab,ebc->eac", P, _expand(Qb, n_elems))
    pos = straight_rods(n_elems, lhat, np.zeros((R, 3)), t)
    vel = rng.normal(0.0, 1e-3, pos.shape)                    # per-node velocities
    return Workload("cfg2", n_elems, _expand(lhat, n_elems), **mat,
                    positions=pos, velocities=vel, directors=dirs,
                    omega=np.zeros((R * N, 3)), clamp=np.full(R, -1, np.int8),
                    gravity=np.array([0.0, 0.0, -9.81]), damping=np.full(R, 0.05),
                    dt=1e-5, n_steps=10000)


def _cfg3(rng, n_rods):
    # 1024^2 filaments x 16 elements, L=0.1, r=1e-3, E=1e6, base clamped with random
    # orientation, tip load N(0,1e-6) per component, damping 0.1, dt=1e-6, 1000 steps.
    R = 1024 * 1024 if n_rods is None else int(n_rods)
    N = 16
    n_elems = np.full(R, N, np.int32)
    lhat = np.full(R, 0.1 / N)
    tip = rng.normal(0.0, 1e-6, (R, 3))                       # per-rod scalars
    mat = _rod_material(R, 1e-3, 1e6)
    Q0 = uniform_so3(rng, R)                                  # per-rod frames
    pos = straight_rods(n_elems, lhat, np.zeros((R, 3)), Q0[:, 2, :])
    dirs = _expand(Q0, n_elems)
    return Workload("cfg3", n_elems, _expand(lhat, n_elems), **mat,
                    positions=pos, velocities=np.zeros_like(pos), directors=dirs,
                    omega=np.zeros((R * N, 3)), clamp=np.zeros(R, np.int8),
                    gravity=np.zeros(3), damping=np.full(R, 0.1), tip_force=tip,
                    dt=1e-6, n_steps=1000)


def _cfg4(rng, n_rods):
    # Active suspension: 65536 rods x 64 elements, L=1, r=0.005, E=1e5, rest curvature
    # kappa0_x = A sin(2 pi (s/L - f t)), A,f ~ U[0.5,2], bases in a 100^3 box, random
    # orientations, damping 0.02, dt=1e-5, 5000 steps.
    R = 65536 if n_rods is None else int(n_rods)
    N = 64
    n_elems = np.full(R, N, np.int32)
    lhat = np.full(R, 1.0 / N)
    A = rng.uniform(0.5, 2.0, R)                              # per-rod scalars
    f = rng.uniform(0.5, 2.0, R)
    base = rng.uniform(0.0, 100.0, (R, 3))
    mat = _rod_material(R, 0.005, 1e5)
    Q0 = uniform_so3(rng, R)                                  # per-rod frames
    pos = straight_rods(n_elems, lhat, base, Q0[:, 2, :])
    return Workload("cfg4", n_elems, _expand(lhat, n_elems), **mat,
                    positions=pos, velocities=np.zeros_like(pos),
                    directors=_expand(Q0, n_elems), omega=np.zeros((R * N, 3)),
                    clamp=np.full(R, -1, np.int8), gravity=np.zeros(3),
                    damping=np.full(R, 0.02), act_A=A, act_f=f, act_L=np.full(R, 1.0),
                    act_component=0, dt=1e-5, n_steps=5000)


def _cfg5(rng, n_rods):
    # Ragged: 262144 rods, N ~ U{8..256}, lhat=0.01, r ~ U[1e-3,1e-2], E log-uniform
    # [1e4,1e7], rest curvature N(0,0.5) per component, half clamped, gravity on,
    # damping 0.05, dt=1e-6, 1000 steps.
    R = 262144 if n_rods is None else int(n_rods)
    n_elems = rng.integers(8, 257, R).astype(np.int32)        # per-rod scalars
    radius = rng.uniform(1e-3, 1e-2, R)
    E = 10.0 ** rng.uniform(4.0, 7.0, R)
    clamped = rng.random(R) < 0.5
    lhat = np.full(R, 0.01)
    mat = _rod_material(R, radius, E)
    Q0 = uniform_so3(rng, R)                                  # per-rod frames
    n_vor = int(n_elems.sum()) - R
    kappa0 = rng.normal(0.0, 0.5, (n_vor, 3))                 # per-element (Voronoi) draws
    pos = straight_rods(n_elems, lhat, np.zeros((R, 3)), Q0[:, 2, :])
    return Workload("cfg5", n_elems, _expand(lhat, n_elems), **mat,
                    positions=pos, velocities=np.zeros_like(pos),
                    directors=_expand(Q0, n_elems), omega=np.zeros((int(n_elems.sum()), 3)),
                    clamp=np.where(clamped, 0, -1).astype(np.int8),
                    gravity=np.array([0.0, 0.0, -9.81]), damping=np.full(R, 0.05),
                    rest_kappa=kappa0, dt=1e-6, n_steps=1000)


def sample_rods(w: Workload, k: int, seed: int = 0) -> np.ndarray:
    """Seeded sample of k rod indices (always includes the first and last rod)."""
    R = w.n_rods
    if k >= R:
        return np.arange(R)
    rng = np.random.Generator(np.random.Philox(SEED_BASE + 1000 + seed))
    mid = rng.choice(np.arange(1, R - 1), size=max(k - 2, 0), replace=False)
    return np.sort(np.concatenate([[0], mid, [R - 1]]))


# ---------------------------------------------------------------------------
# NEXT-2: magnetic cilia.  Not a BASELINE config; parameters are
# a synthetic stand-in (the paper's cilia parameters live in its missing supplement).
# ---------------------------------------------------------------------------
CILIA = dict(N=20, L=0.01, radius=5e-4, E=1e5, rho=1000.0, spacing=3e-3, b=0.02,
             theta_lin=0.1, beat_hz=10.0, wavelength_cols=8, damping=50.0, dt=2e-5)


def _cilia(name, n_rods):
    """Clamped (s = 0) cilia standing along +z on a square grid; magnetisation per unit length
    of magnitude m (set so the quasi-static tip angle m b L^2 / (2 E I) is theta_lin) at an angle
    psi = 2 pi ix / wavelength_cols from d3 towards d1 (a programmed metachronal phase);
    homogeneous field b(t) = b (cos, 0, -sin)(2 pi f t) rotating about lab y."""
    c = CILIA
    if name == "cilia8":
        nx = ny = 8
    else:
        nx, ny = 335, 334          # 111,890 sites; the first 111,797 are used
    R_full = 111797 if name == "ciliafarm" else nx * ny
    R = R_full if n_rods is None else int(n_rods)
    N = c["N"]
    ids = np.arange(R)
    ix, iy = ids % nx, ids // nx
    n_elems = np.full(R, N, np.int32)
    lhat = np.full(R, c["L"] / N)
    mat = _rod_material(R, c["radius"], c["E"], rho=c["rho"])
    base = np.stack([ix * c["spacing"], iy * c["spacing"], np.zeros(R)], axis=1)
    d3 = np.tile([0.0, 0.0, 1.0], (R, 1))
    pos = straight_rods(n_elems, lhat, base, d3)
    EI = c["E"] * mat["I1"][0]
    m = c["theta_lin"] * 2.0 * EI / (c["b"] * c["L"] ** 2)
    psi = 2.0 * math.pi * ix / c["wavelength_cols"]
    mag_rod = np.stack([m * np.sin(psi), np.zeros(R), m * np.cos(psi)], axis=1)
    return Workload(name, n_elems, _expand(lhat, n_elems), **mat, positions=pos,
                    velocities=np.zeros_like(pos), directors=np.tile(np.eye(3), (R * N, 1, 1)),
                    omega=np.zeros((R * N, 3)), clamp=np.zeros(R, np.int8), gravity=np.zeros(3),
                    damping=np.full(R, c["damping"]), magnetization=_expand(mag_rod, n_elems),
                    b_field=np.array([c["b"], 0.0, 0.0]), b_omega=2.0 * math.pi * c["beat_hz"],
                    b_axis=np.array([0.0, 1.0, 0.0]), dt=c["dt"], n_steps=20000)


# ---------------------------------------------------------------------------
# NEXT-4: contact stand-in for the fibrous-packing study (1536 filaments,
# frictional rod-rod and rod-boundary contact, HHG broad phase).  The paper's packing parameters
# live in its missing supplement; this is a synthetic recipe with cfg3's rods (L = 0.1, r = 1e-3,
# E = 1e6, 16 elements): stacks of crossed layers ("woven mats") resting on a floor, every layer
# pressed into the next by a small overlap, so contacts exist from the first step.
# ---------------------------------------------------------------------------
FIBRES = dict(N=16, L=0.1, radius=1e-3, E=1e6, rho=1000.0, per_layer=16, layers=16, overlap=2e-6,
              jitter_angle=0.02, v_sd=1e-4, damping=0.1, gamma_n=0.02, mu=0.4, v_stick=1e-3,
              dt=1e-6)


def _fibres(n_rods):
    """Rods fill stacks (layer by layer) of `layers` x `per_layer` rods; stacks sit on a square
    grid of pitch 1.2 L.  Layer k of a stack: rods along x (k even) or y (k odd), evenly spaced
    across the stack's L x L footprint, in-plane angle jitter U(-0.02, 0.02) rad, height
    z_k = r - overlap/2 + k (2r - overlap) + U(-overlap/4, overlap/4) (the bottom layer presses into
    the floor z = 0 by overlap/2 +- overlap/4); velocities N(0, 1e-4) per component.  Default full size: 256 stacks
    of 16 x 16 rods = 65,536 rods x 16 elements (1,048,576 elements, cfg3's element count)."""
    c = FIBRES
    rng = np.random.Generator(np.random.Philox(SEED_BASE + 6))
    per_stack = c["layers"] * c["per_layer"]
    R = 256 * per_stack if n_rods is None else int(n_rods)
    N, L, r, ov = c["N"], c["L"], c["radius"], c["overlap"]
    ids = np.arange(R)
    stack, k, j = ids // per_stack, (ids % per_stack) // c["per_layer"], ids % c["per_layer"]
    G = max(1, int(math.ceil(math.sqrt(max(1, (R + per_stack - 1) // per_stack)))))
    ox, oy = (stack % G) * 1.2 * L, (stack // G) * 1.2 * L
    phi = np.where(k % 2 == 0, 0.0, 0.5 * math.pi) + rng.uniform(-c["jitter_angle"], c["jitter_angle"], R)
    z = r - ov / 2 + k * (2 * r - ov) + rng.uniform(-ov / 4, ov / 4, R)
    across = (j + 0.5) * L / c["per_layer"]
    cx = ox + np.where(k % 2 == 0, 0.5 * L, across)
    cy = oy + np.where(k % 2 == 0, across, 0.5 * L)
    d3 = np.stack([np.cos(phi), np.sin(phi), np.zeros(R)], axis=1)
    base = np.stack([cx, cy, z], axis=1) - 0.5 * L * d3
    n_elems = np.full(R, N, np.int32)
    lhat = np.full(R, L / N)
    frames = complete_frame(d3)
    pos = straight_rods(n_elems, lhat, base, d3)
    vel = rng.normal(0.0, c["v_sd"], pos.shape)
    mat = _rod_material(R, r, c["E"], rho=c["rho"])
    contact = Contact(k_n=0.0, gamma_n=c["gamma_n"], mu_s=c["mu"], mu_k=c["mu"], v_stick=c["v_stick"],
                      exclude=2, plane_n=np.array([0.0, 0.0, 1.0]), plane_d=0.0)
    return Workload("fibres", n_elems, _expand(lhat, n_elems), **mat, positions=pos, velocities=vel,
                    directors=_expand(frames, n_elems), omega=np.zeros((R * N, 3)),
                    clamp=np.full(R, -1, np.int8), gravity=np.array([0.0, 0.0, -9.81]),
                    damping=np.full(R, c["damping"]), dt=c["dt"], n_steps=1000, contact=contact)
