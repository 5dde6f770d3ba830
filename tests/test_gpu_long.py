"""Long rods (more than ER_TILE_MAX_ELEMS = 511 elements): each rod is advanced by a thread-block
cluster, one CTA per 256-slot segment, neighbour data crossing segments through distributed
shared memory.  Parity against the oracle (which has no length limit), alone and mixed with tile
rods, with every load type, plus layout round trips, temporal blocking and diagnostics."""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import TOL_1000, TOL_1STEP, assert_directors_round_trip, assert_parity
from rodkit import concat, rod

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


def perturbed(ns, seed=11, clamp=None, tip=False):
    """Rods of the given lengths (L = 0.01 N, r = 5 mm, E = 1e6), random orientation, directors
    perturbed element by element (angle <= 0.05), random v and w: a non-degenerate state."""
    rng = np.random.default_rng(seed)
    ws = []
    for q, N in enumerate(ns):
        Q0 = W.uniform_so3(rng, 1)[0]
        ws.append(rod(N=N, L=0.01 * N, r=0.005, E=1e6, Q=Q0, base=tuple(rng.uniform(-1, 1, 3)),
                      clamp=-1 if clamp is None else clamp[q], tip=(rng.normal(0, 1e-4, 3) if tip else None),
                      nu=0.05, g=(0, 0, -9.81), dt=1e-5))
    w = concat(ws)
    if tip:
        w.tip_force = np.stack([x.tip_force[0] for x in ws])
    E = w.n_elems_total
    ax = rng.standard_normal((E, 3))
    ang = rng.uniform(0, 0.05, E)
    R = W.quat_to_rows(W.axis_angle_quat(ax, ang))
    w.directors = np.einsum("eab,ebc->eac", R, w.directors)
    w.velocities = rng.normal(0, 1e-3, w.velocities.shape)
    w.omega = rng.normal(0, 1e-2, w.omega.shape)
    return w


def run_gpu(er, w, n_steps, **kw):
    with er.RodBatch(w, **kw) as b:
        b.step(n_steps, w.dt)
        return b.get_state()


def run_orc(orc, w, n_steps):
    st, s, bad, bits = orc.step(w, n_steps=n_steps)
    assert s == 0, (bad, bits)
    return (st.positions, st.velocities, st.directors, st.omega), st.t


@pytest.mark.parametrize("ns", [[600], [256, 1023, 5, 700], [2047]])
def test_long_rods_parity(er, orc, ns):
    w = perturbed(ns)
    g = run_gpu(er, w, 1)
    o, t = run_orc(orc, w, 1)
    assert g[4] == t
    assert_parity(w, g[:4], o, TOL_1STEP, raw=("r", "v", "Q", "w"), label=f"{ns} 1 step")
    g = run_gpu(er, w, 300)
    o, _ = run_orc(orc, w, 300)
    assert_parity(w, g[:4], o, TOL_1000, raw=("r", "Q"), label=f"{ns} 300 steps")


def test_long_rod_loads_and_bcs(er, orc):
    """Clamps at either end, tip loads, actuation, static rest curvature, general (non-uniform)
    rest lengths on long rods next to short ones."""
    ns = [900, 12, 530, 1200]
    w = perturbed(ns, seed=3, clamp=[0, -1, 1, 0], tip=True)
    rng = np.random.default_rng(4)
    lh = w.rest_lengths.copy()
    lh[w.elem_offsets()[3]:] *= 1.0 + 0.1 * rng.uniform(-1, 1, w.n_elems[3])   # rod 3 non-uniform
    w = dataclasses.replace(w, rest_lengths=lh, rest_kappa=rng.normal(0, 0.5, (w.n_voronoi_total, 3)),
                            act_A=np.array([1.0, 0.0, 0.5, 2.0]), act_f=np.array([1.0, 1.0, 2.0, 0.5]),
                            act_L=0.01 * np.array(ns, float), act_component=1)
    g = run_gpu(er, w, 1)
    o, _ = run_orc(orc, w, 1)
    assert_parity(w, g[:4], o, TOL_1STEP, raw=("r", "v", "Q"), label="loads 1 step")
    g = run_gpu(er, w, 200)
    o, _ = run_orc(orc, w, 200)
    assert_parity(w, g[:4], o, TOL_1000, raw=("r", "Q"), label="loads 200 steps")


def test_long_rod_layout_and_modes(er, monkeypatch):
    """Create / get_state round trip bitwise; temporal blocking, the staged kernel mode and the
    non-persistent cluster kernel (ER_LONG_SIMPLE) give the same trajectory bitwise."""
    w = perturbed([1500, 40, 513, 3])
    with er.RodBatch(w) as b:
        pos, vel, dirs, om, _ = b.get_state()
    for x, y in ((pos, w.positions), (vel, w.velocities), (om, w.omega)):
        assert np.array_equal(x, y)
    assert_directors_round_trip(dirs, w.directors)
    ref = run_gpu(er, w, 24)
    for opt, val in ((er.ER_OPT_STEPS_PER_LAUNCH, 8), (er.ER_OPT_KERNEL, 1)):
        with er.RodBatch(w) as b:
            b.set_option(opt, val)
            b.step(24, w.dt)
            out = b.get_state()
        for x, y in zip(out[:4], ref[:4]):
            assert np.array_equal(x, y)
    monkeypatch.setenv("ER_LONG_SIMPLE", "1")
    out = run_gpu(er, w, 24)
    for x, y in zip(out[:4], ref[:4]):
        assert np.array_equal(x, y)


def test_long_rod_diagnostics(er, orc):
    w = perturbed([800, 300, 1100])
    with er.RodBatch(w) as b:
        b.step(5, w.dt)
        d = b.diagnostics()
    st, _, _, _ = orc.step(w, n_steps=5)
    ref = orc.energy(w, st)
    # the tolerances of test_gpu_parity.py::test_diagnostics_match_oracle (sums with cancellation)
    mass, vmax = ref[10], ref[9]
    scale = max(np.max(np.abs(ref[:6])), mass * np.linalg.norm(w.gravity) * np.max(np.abs(st.positions)))
    assert np.all(np.abs(d[:6] - ref[:6]) <= 1e-10 * np.abs(ref[:6]) + 1e-12 * scale), (d, ref)
    assert np.all(np.abs(d[6:9] - ref[6:9]) <= 1e-12 * mass * vmax), (d, ref)
    assert np.isclose(d[9], ref[9], rtol=1e-12) and np.isclose(d[10], ref[10], rtol=1e-13) and d[11] == ref[11]


def test_longest_rod(er):
    w = perturbed([er.ER_MAX_ELEMS_PER_ROD])                      # 16 segments: the largest cluster
    g = run_gpu(er, w, 2)
    assert all(np.all(np.isfinite(x)) for x in g[:4])
    too_long = perturbed([er.ER_MAX_ELEMS_PER_ROD + 1])
    with pytest.raises(er.ErError):
        er.RodBatch(too_long)


def test_long_rods_in_contact(er, orc):
    """A 700-element rod lying across short rods on a floor: contact forces reach the long rod's
    segments (cluster kernel, contact mode) exactly as the oracle's exhaustive search says; the
    fused and staged contact paths agree bitwise."""
    N, lh, r = 700, 0.002, 0.004
    L = N * lh
    ws = [rod(N=N, L=L, r=r, Q=np.array([[0, 0, -1.0], [0, 1.0, 0], [1.0, 0, 0]]), base=(-L / 2, 0.0, 3 * r - 2e-6),
              g=(0, 0, -9.81), nu=1.0, dt=2e-6)]
    for k in range(6):                                   # short rods along y, under the long rod
        x = -0.5 + 0.2 * k
        ws.append(rod(N=10, L=0.1, r=r, Q=np.array([[1.0, 0, 0], [0, 0, -1.0], [0, 1.0, 0]]),
                      base=(x, -0.05, r - 1e-6), g=(0, 0, -9.81), nu=1.0, dt=2e-6))
    w = concat(ws)
    w.velocities = np.random.default_rng(2).normal(0, 1e-3, w.velocities.shape)
    w.contact = W.Contact(k_n=2e3, gamma_n=0.05, mu_s=0.3, mu_k=0.3, v_stick=1e-3,
                          plane_n=np.array([0, 0, 1.0]), plane_d=0.0)
    with er.RodBatch(w) as b:
        b.step(1, w.dt)
        g1 = b.get_state()
        st = b.contact_stats()
    assert st.contacts >= 6 and st.plane_contacts > 0
    o, _ = run_orc(orc, w, 1)
    assert_parity(w, g1[:4], o, TOL_1STEP, raw=("r", "v", "Q"), label="long rod contact 1 step")
    out = []
    for kernel in (0, 1):
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_KERNEL, kernel)
            b.step(150, w.dt)
            out.append(b.get_state())
    for x, y in zip(out[0][:4], out[1][:4]):
        assert np.array_equal(x, y)
    o, _ = run_orc(orc, w, 150)
    assert_parity(w, out[0][:4], o, TOL_1000, raw=("r", "Q"), label="long rod contact 150 steps")


def test_long_rod_batch_full_size_sampled(er, orc):
    """16,384 rods x 1000 elements (the long-rod timing workload of tools/long_rod_time.py, 16.4 M
    elements: 4-CTA clusters), 200 steps on the GPU; the oracle re-runs 8 sampled rods."""
    R, N = 16384, 1000
    n = np.full(R, N, np.int32)
    lh = np.full(R, 0.00625)
    mat = W._rod_material(R, 1e-3, 1e6)
    rng = np.random.default_rng(0)
    Q0 = W.uniform_so3(rng, R)
    pos = W.straight_rods(n, lh, np.zeros((R, 3)), Q0[:, 2, :])
    w = W.Workload("long", n, W._expand(lh, n), **mat, positions=pos, velocities=np.zeros_like(pos),
                   directors=W._expand(Q0, n), omega=np.zeros((R * N, 3)), clamp=np.zeros(R, np.int8),
                   gravity=np.zeros(3), damping=np.full(R, 0.1), tip_force=rng.normal(0, 1e-6, (R, 3)), dt=1e-6)
    g = run_gpu(er, w, 200)
    rods = np.array([0, 1, 777, 5000, 9999, 12345, R - 2, R - 1])
    ws = w.subset(rods)
    no, eo = w.node_offsets(), w.elem_offsets()
    nidx = np.concatenate([np.arange(no[r], no[r + 1]) for r in rods])
    eidx = np.concatenate([np.arange(eo[r], eo[r + 1]) for r in rods])
    o, _ = run_orc(orc, ws, 200)
    assert_parity(ws, (g[0][nidx], g[1][nidx], g[2][eidx], g[3][eidx]), o, TOL_1000, raw=("r", "Q"),
                  label="16384 x 1000 sampled, 200 steps")
