"""GPU parity of the contact path (DESIGN §3 #27): HHG broad phase + exact
segment-segment narrow phase + penalty / regularised-Coulomb law on the GPU vs the oracle's
exhaustive O(E^2) search on the same seeded inputs.

Rods that touch are no longer independent, so full-size parity samples whole *stacks* of the
`fibres` workload: its stacks sit 0.2 L apart and never touch, so one stack is an independent
sub-problem the oracle can run on its own.
"""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import TOL_1000, TOL_1STEP, assert_parity, errors
from rodkit import concat, rod

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


def run_gpu(er, w, n_steps, **contact_kw):
    with er.RodBatch(w, apply_bc_forcing=True) as b:
        if contact_kw:
            b.set_contact(w.contact, **contact_kw)
        b.step(n_steps, w.dt)
        pos, vel, dirs, om, t = b.get_state()
        stats = b.contact_stats()
    return (pos, vel, dirs, om), t, stats


def run_orc(orc, w, n_steps):
    st, s, bad, bits = orc.step(w, n_steps=n_steps)
    assert s == 0, (bad, bits)
    return (st.positions, st.velocities, st.directors, st.omega), st.t


def mixed_radii(n_rods=64):
    """fibres with every third layer of contact radius 2.5 mm (the others 1 mm), the layers
    re-stacked so that neighbouring layers overlap by the recipe's 2 um: two populated HHG
    levels, so thin-thick pairs cross levels (cross-level records) and thin-thin pairs do not.
    (Overlapping the fat rods by millimetres instead makes the problem explode: a 1-ulp input
    change then moves the oracle's own result by 1e-5 within 300 steps.)"""
    w = W.make("fibres", n_rods=n_rods)
    c = W.FIBRES
    k = (np.arange(w.n_rods) % (c["layers"] * c["per_layer"])) // c["per_layer"]
    r_layer = np.where(np.arange(c["layers"]) % 3 == 2, 2.5e-3, 1e-3)
    z_layer = np.cumsum(np.r_[r_layer[0] - c["overlap"] / 2, r_layer[:-1] + r_layer[1:] - c["overlap"]])
    z_old = c["radius"] - c["overlap"] / 2 + k * (2 * c["radius"] - c["overlap"])
    pos = w.positions.copy()
    pos[:, 2] += np.repeat(z_layer[k] - z_old, w.n_elems + 1)
    return dataclasses.replace(w, positions=pos,
                               contact=dataclasses.replace(w.contact, radius=r_layer[k].copy()))


def test_fibres_one_step(er, orc):
    w = W.make("fibres", n_rods=64)                      # 4 crossed layers, 1024 elements
    g, tg, st = run_gpu(er, w, 1)
    o, to = run_orc(orc, w, 1)
    assert tg == to
    assert_parity(w, g, o, TOL_1STEP, raw=("r", "v", "Q"), label="fibres 1 step")
    # same contact set as the oracle's exhaustive search at the drift-1 configuration
    half = w.positions + 0.5 * w.dt * w.velocities
    pairs, _ = orc.contact_pairs(w, half)
    assert st.contacts == len(pairs) > 500
    assert st.plane_contacts == np.count_nonzero(half[:, 2] < 1e-3) == 16 * 17   # bottom layer on the floor
    assert st.candidates >= st.contacts


def test_fibres_1000_steps(er, orc):
    w = W.make("fibres", n_rods=32)
    g, _, st = run_gpu(er, w, 1000)
    o, _ = run_orc(orc, w, 1000)
    e = assert_parity(w, g, o, TOL_1000, raw=("r", "Q"), label="fibres 1000 steps")
    assert st.contacts > 0


def test_cross_level_pairs(er, orc):
    w = mixed_radii()
    g, _, st = run_gpu(er, w, 1)
    assert st.n_levels >= 2 and bin(st.level_mask).count("1") == 2
    assert st.cross_level > 0 and st.pool_used == st.cross_level
    o, _ = run_orc(orc, w, 1)
    assert_parity(w, g, o, TOL_1STEP, raw=("r", "v", "Q"), label="mixed radii 1 step")
    g, _, _ = run_gpu(er, w, 300)
    o, _ = run_orc(orc, w, 300)
    assert_parity(w, g, o, TOL_1000, raw=("r", "Q"), label="mixed radii 300 steps")


def test_single_level_grid_gives_same_forces(er):
    """The HHG level split changes which proxy evaluates a pair, never the result: one level
    (cells for the largest element) vs the automatic hierarchy agree to round-off."""
    w = mixed_radii()
    a, _, sa = run_gpu(er, w, 20)
    b, _, sb = run_gpu(er, w, 20, cell0=0.02, n_levels=1)
    assert sb.cross_level == 0 and sa.cross_level > 0
    assert sa.contacts == sb.contacts
    e = errors(w, a, b)
    assert max(v for k, v in e.items() if not k.endswith("_raw")) < 1e-13, e


def test_deterministic(er):
    w = mixed_radii()
    a, _, _ = run_gpu(er, w, 50)
    b, _, _ = run_gpu(er, w, 50)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_head_on_impact_momentum(er, orc):
    """Two crossing rods, one falling onto the other, no gravity / damping / plane: the contact
    forces are equal and opposite, so total momentum is conserved to round-off."""
    L, N, r = 0.4, 8, 0.01
    lh = L / N
    A = rod(N=N, L=L, r=r, Q=np.array([[0, 0, -1.0], [0, 1.0, 0], [1.0, 0, 0]]), base=(-L / 2 - lh / 2, 0, 0))
    d = np.array([0.5, np.sqrt(0.75), 0.0])
    Qb = np.stack([[0, 0, 1.0], np.cross(d, [0, 0, 1.0]), d])
    B = rod(N=N, L=L, r=r, Q=Qb, base=tuple(-(L / 2 + lh / 2) * d + np.array([0, 0, 2 * r + 5e-4])))
    w = concat([A, B])
    w.contact = W.Contact(k_n=5e3, gamma_n=2.0, mu_s=0.3, mu_k=0.2)
    w.velocities[9:, 2] = -0.5
    w.dt = 1e-6
    g, _, _ = run_gpu(er, w, 3000)
    o, _ = run_orc(orc, w, 3000)
    assert_parity(w, g, o, TOL_1000, raw=("r", "v", "Q"), label="impact 3000 steps")
    m = w.density[0] * w.area[0] * lh * np.r_[0.5, np.ones(N - 1), 0.5]
    P0 = (np.r_[m, m][:, None] * w.velocities).sum(0)
    P1 = (np.r_[m, m][:, None] * g[1]).sum(0)
    assert np.allclose(P1, P0, rtol=0, atol=1e-13)
    assert g[1][9:, 2].mean() > -0.5


def test_grid_overflow_faults(er):
    """An element wider than the top HHG level cannot be binned: ER_F_CONTACT, rod id reported."""
    w = W.make("fibres", n_rods=16)
    with er.RodBatch(w) as b:
        b.set_contact(w.contact, cell0=1e-3, n_levels=1)
        with pytest.raises(er.ErError) as ei:
            b.step(1, w.dt)
        rod_id, bits = b.fault()
        assert ei.value.status == er.ER_EUNSTABLE and bits & er.ER_F_CONTACT and rod_id == 0


def test_full_size_sampled_stacks(er, orc):
    """Full fibres workload (65,536 rods, 1,048,576 elements, bench.py's launch configuration):
    after 1 and 5 steps two sampled stacks match the oracle run on those stacks alone."""
    w = W.make("fibres")
    per_stack = W.FIBRES["layers"] * W.FIBRES["per_layer"]
    with er.RodBatch(w) as b:
        b.step(1, w.dt)
        s1 = b.get_state()
        st1 = b.contact_stats()
        b.step(4, w.dt)
        s5 = b.get_state()
    assert st1.contacts > 200_000
    no, eo = w.node_offsets(), w.elem_offsets()
    for stack in (0, 173):
        rods = np.arange(stack * per_stack, (stack + 1) * per_stack)
        ws = w.subset(rods)
        nsl = slice(no[rods[0]], no[rods[-1] + 1])
        esl = slice(eo[rods[0]], eo[rods[-1] + 1])
        for s, n, tol in ((s1, 1, TOL_1STEP), (s5, 5, TOL_1STEP * 10)):
            g = (s[0][nsl], s[1][nsl], s[2][esl], s[3][esl])
            o, _ = run_orc(orc, ws, n)
            assert_parity(ws, g, o, tol, raw=("r", "Q"), label=f"stack {stack} after {n} steps")


def test_verlet_skin_changes_nothing(er, orc):
    """Candidate lists are reused until a node moves skin/2: a tiny skin (a rebuild almost every
    step) and a large one give the same trajectory to round-off, and both match the oracle."""
    w = mixed_radii()
    w.velocities = w.velocities * 300.0                  # ~3 cm/s: 3e-8 m per step
    runs = {}
    for skin in (1e-7, 0.0, 2e-3):
        with er.RodBatch(w) as b:
            b.set_contact(w.contact, skin=skin)
            b.step(200, w.dt)
            runs[skin] = (b.get_state()[:4], b.contact_stats())
    assert runs[1e-7][1].builds > 50 and runs[2e-3][1].builds == 1
    for skin in (0.0, 2e-3):
        e = errors(w, runs[1e-7][0], runs[skin][0])
        assert max(v for k, v in e.items() if not k.endswith("_raw")) < 1e-13, (skin, e)
    o, _ = run_orc(orc, w, 200)
    assert_parity(w, runs[0.0][0], o, TOL_1000, raw=("r", "Q"), label="moving mixed radii 200 steps")


def test_set_state_forces_rebuild(er, orc):
    """Teleporting rods with er_set_state invalidates the lists: the next step rebuilds."""
    w = W.make("fibres", n_rods=32)
    with er.RodBatch(w) as b:
        b.step(3, w.dt)
        n0 = b.contact_stats().builds
        pos = w.positions.copy()
        pos[:, 0] += 0.5                                # every rod moved by 0.5 m: no stale pair
        b.set_state(positions=pos, velocities=w.velocities, directors=w.directors, omega=w.omega, t=0.0)
        b.step(1, w.dt)
        st = b.contact_stats()
        g = b.get_state()[:4]
    assert st.builds == n0 + 1
    w2 = dataclasses.replace(w, positions=pos)
    o, _ = run_orc(orc, w2, 1)
    assert_parity(w2, g, o, TOL_1STEP, raw=("r", "v", "Q"), label="after set_state")


def test_fused_equals_staged(er):
    """The fused contact step (one persistent launch: kick + drift-2 + next drift-1 + node
    records) is bitwise the staged one (drift | contact | dynamics | drift as separate kernels)."""
    w = mixed_radii()
    out = []
    for kernel in (0, 1):
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_KERNEL, kernel)
            b.step(37, w.dt)
            b.step(13, w.dt)
            out.append(b.get_state())
    for x, y in zip(out[0], out[1]):
        assert np.array_equal(x, y)


def test_graph_equals_plain_launches(er, monkeypatch):
    """The per-step contact graph (conditional list build / long-list pass decided on the device)
    is bitwise the plain launch sequence; rebuilds happen inside the graph."""
    w = mixed_radii()
    w.velocities = w.velocities * 300.0
    out = []
    for no_graph in (False, True):
        if no_graph:
            monkeypatch.setenv("ER_NO_GRAPH", "1")
        with er.RodBatch(w) as b:
            b.set_contact(w.contact, skin=2e-7)
            b.step(60, w.dt)
            out.append((b.get_state(), b.contact_stats().builds))
    assert out[0][1] == out[1][1] > 10
    for x, y in zip(out[0][0], out[1][0]):
        assert np.array_equal(x, y)


def edge_case_workload():
    """Single-element rods (both nodes on one element: the half-space law on two nodes), clamped
    rods, non-uniform rest lengths and per-rod radii together, against the oracle.  Each rod gets
    its own height (7.2 mm apart, radii 3-4.5 mm: overlaps below 1.8 mm, so the problem stays
    well conditioned over the run): crossing rods at the SAME height have intersecting axes, where
    the contact normal (pa - pb)/|pa - pb| is undefined -- round-off then decides it, on both
    sides differently (a degenerate configuration of the capsule model, not a parity case)."""
    rng = np.random.default_rng(5)
    ws = []
    for q in range(12):
        N = [1, 2, 5][q % 3]
        ang = rng.uniform(0, np.pi)
        d = np.array([np.cos(ang), np.sin(ang), 0.0])
        Q = np.stack([[0, 0, 1.0], np.cross(d, [0, 0, 1.0]), d])
        base = (rng.uniform(-0.02, 0.02) - 0.02 * d[0], rng.uniform(-0.02, 0.02) - 0.02 * d[1], 0.0028 + 0.0072 * q)
        ws.append(rod(N=N, L=0.04, r=0.004, Q=Q, base=base, clamp=0 if q % 5 == 0 else -1, g=(0, 0, -9.81),
                      nu=2.0, dt=2e-6))
    w = concat(ws)
    lh = w.rest_lengths.copy()
    lh *= 1.0 + 0.05 * np.sin(np.arange(len(lh)))          # non-uniform rest lengths ("general" rods)
    w = dataclasses.replace(w, rest_lengths=lh)
    w.velocities = rng.normal(0, 0.01, w.velocities.shape)
    w.contact = W.Contact(k_n=500.0, gamma_n=0.1, mu_s=0.4, mu_k=0.3, v_stick=1e-3,
                          radius=rng.uniform(0.003, 0.0045, w.n_rods), plane_n=np.array([0, 0, 1.0]), plane_d=0.0)
    return w


def test_contact_edge_cases(er, orc):
    w = edge_case_workload()
    g, _, st = run_gpu(er, w, 1)
    o, _ = run_orc(orc, w, 1)
    assert_parity(w, g, o, TOL_1STEP, raw=("r", "v", "Q"), label="edge cases 1 step")
    assert st.contacts > 0 and st.plane_contacts > 0
    g, _, _ = run_gpu(er, w, 500)
    o, _ = run_orc(orc, w, 500)
    assert_parity(w, g, o, TOL_1000, raw=("r", "Q"), label="edge cases 500 steps")


def test_contact_empty_and_disable(er):
    w = W.make("fibres", n_rods=16)
    with er.RodBatch(w) as b:
        b.step(3, w.dt)
        b.set_contact(None)                              # back to independent rods
        b.step(3, w.dt)
        assert b.contact_stats().contacts == 0
    e = dataclasses.replace(W.make("fibres", n_rods=16).subset(np.arange(0)), contact=w.contact)
    with er.RodBatch(e) as b:
        b.step(5, w.dt)
        assert b.contact_stats().contacts == 0
