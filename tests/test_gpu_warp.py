"""The warp-local step kernel (csrc/er_warp.cu) for batches of equal-length short rods.

Rods of ER_WARP_MIN_N..32 elements run one rod per N lanes of a warp, with warp-shuffle exchanges
and no CTA barriers.  Its physics is the tile kernel's, so both must give the same
trajectory (ER_NO_WARP=1 selects the tile kernel on the same inputs), and both must match the oracle
(tests/parity.py gates).  Covered: rods of 4..32 elements (several per warp, one per warp, padded
lanes), clamps at either end, tip loads, actuation, static rest curvature, per-element material,
sigma0 / magnetic / muscle / external loads, temporal blocking, step graphs, faults, diagnostics,
and BASELINE cfg3 at full size.
"""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import TOL_1000, TOL_1STEP, assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


@pytest.fixture(autouse=True)
def force_warp_layout(monkeypatch):
    """The warp layout is chosen for large batches only; these tests use small ones."""
    monkeypatch.setenv("ER_WARP", "1")


def run(er, w, n_steps, warp=True, monkeypatch=None, spl=1, dt=None, sweeps=1):
    if not warp:
        monkeypatch.setenv("ER_NO_WARP", "1")
    try:
        with er.RodBatch(w) as b:
            info = b.info()
            assert (info.warp_rod_elems > 0) == warp, (info.warp_rod_elems, warp)
            b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, sweeps)
            if spl != 1:
                b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
            b.step(n_steps, w.dt if dt is None else dt)
            out = b.get_state()
            d = b.diagnostics()
    finally:
        if not warp:
            monkeypatch.delenv("ER_NO_WARP")
    return out, d


def uniform_batch(N, R, seed, clamp_mix=True, tip=True):
    """R rods of N elements: random frames, perturbed directors and velocities, clamps at s = 0 /
    s = L / free, tip loads (so every term of the step is active)."""
    import scipy.linalg as sla
    rng = np.random.default_rng(seed)
    w = W.make("cfg3", n_rods=R)
    lh = 0.1 / N
    n = np.full(R, N, np.int32)
    base = rng.uniform(-1, 1, (R, 3))
    frames = np.stack([sla.expm(np.cross(np.eye(3), rng.standard_normal(3))) for _ in range(R)])
    pos = W.straight_rods(n, np.full(R * N, lh), base, frames[:, 2, :])
    dirs = np.repeat(frames, N, axis=0)
    K = lambda v: np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])
    dirs = np.stack([sla.expm(K(rng.standard_normal(3) * 0.02)) for _ in range(R * N)]) @ dirs
    mat = W._rod_material(R, 1e-3, 10 ** rng.uniform(5, 6.5, R))
    clamp = rng.integers(-1, 2, R).astype(np.int8) if clamp_mix else np.full(R, -1, np.int8)
    w = dataclasses.replace(
        w, name=f"u{N}", n_elems=n, rest_lengths=np.full(R * N, lh), **mat, positions=pos,
        velocities=rng.standard_normal(pos.shape) * 1e-3, directors=dirs,
        omega=rng.standard_normal((R * N, 3)) * 0.1, clamp=clamp, gravity=np.array([0.0, -1.0, -9.81]),
        damping=rng.uniform(0, 0.2, R), tip_force=rng.standard_normal((R, 3)) * 1e-6 if tip else None,
        dt=1e-6)
    return w


def same(a, b, rtol=0.0):
    for x, y in zip(a, b):
        x, y = np.asarray(x), np.asarray(y)
        if rtol == 0.0:
            assert np.array_equal(x, y)
        else:
            assert np.max(np.abs(x - y), initial=0.0) <= rtol * max(1.0, np.max(np.abs(y), initial=0.0))


@pytest.mark.parametrize("N,R", [(16, 600), (4, 300), (5, 333), (15, 250), (17, 200), (31, 100), (32, 90),
                                 (33, 90), (40, 80), (64, 70)])
def test_warp_equals_tile_kernel(er, monkeypatch, N, R):
    w = uniform_batch(N, R, seed=N)
    a, da = run(er, w, 50)
    b, db = run(er, w, 50, warp=False, monkeypatch=monkeypatch)
    same(a, b)
    # diagnostics sum per tile (the two kernels tile the batch differently): equal up to summation order
    assert np.allclose(da, db, rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("N", [16, 7, 64, 45])
def test_warp_parity_vs_oracle(er, orc, N):
    w = uniform_batch(N, 300, seed=100 + N)
    for n_steps, tol in ((1, TOL_1STEP), (1000, TOL_1000)):
        g, _ = run(er, w, n_steps)
        st, s, bad, bits = orc.step(w, n_steps=n_steps)
        assert s == 0
        assert_parity(w, g, (st.positions, st.velocities, st.directors, st.omega), tol, raw=("r", "v", "Q", "w"),
                      label=f"warp kernel N={N} x{n_steps}")


def test_warp_features_equal_tile_kernel(er, monkeypatch):
    """Actuation, static rest curvature, per-element material (general rods), sigma0, magnetisation,
    muscle wave and user external loads on the warp kernel vs the tile kernel."""
    w = uniform_batch(12, 200, seed=7)
    rng = np.random.default_rng(9)
    R, E = w.n_rods, w.n_elems_total
    w.act_A, w.act_f, w.act_L = rng.uniform(0.5, 2, R), rng.uniform(0.5, 2, R), np.full(R, 0.1)
    w.act_component = 1
    out_act = [run(er, w, 40)[0], run(er, w, 40, warp=False, monkeypatch=monkeypatch)[0]]
    same(*out_act)
    w.rest_kappa = rng.standard_normal((w.n_voronoi_total, 3)) * 0.5
    same(run(er, w, 40)[0], run(er, w, 40, warp=False, monkeypatch=monkeypatch)[0])
    rod_of = np.repeat(np.arange(R), w.n_elems)
    for name in ("density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c"):
        setattr(w, name, getattr(w, name)[rod_of] * rng.uniform(0.9, 1.1, E))
    w.rest_lengths = w.rest_lengths * rng.uniform(0.95, 1.05, E)
    w.rest_sigma = rng.standard_normal((E, 3)) * 1e-4
    w.magnetization = rng.standard_normal((E, 3)) * 1e-4
    w.b_field, w.b_omega = np.array([1e-2, 0.0, 5e-3]), 30.0
    w.musc_A, w.musc_T = rng.uniform(1e-9, 1e-8, R), rng.uniform(0.5, 2, R)
    w.musc_lambda, w.musc_phi = rng.uniform(0.05, 0.1, R), rng.uniform(0, 6, R)
    w.musc_component = 2
    w.ext_force = rng.standard_normal((w.n_nodes_total, 3)) * 1e-7
    w.ext_couple = rng.standard_normal((E, 3)) * 1e-10
    a, da = run(er, w, 40)
    b, db = run(er, w, 40, warp=False, monkeypatch=monkeypatch)
    same(a, b)


def test_warp_features_parity(er, orc):
    w = uniform_batch(9, 120, seed=21)
    rng = np.random.default_rng(22)
    R, E = w.n_rods, w.n_elems_total
    w.act_A, w.act_f, w.act_L = rng.uniform(0.5, 2, R), rng.uniform(0.5, 2, R), np.full(R, 0.1)
    w.rest_kappa = rng.standard_normal((w.n_voronoi_total, 3)) * 0.5
    w.rest_sigma = rng.standard_normal((E, 3)) * 1e-4
    w.ext_couple = rng.standard_normal((E, 3)) * 1e-10
    for n_steps, tol in ((1, TOL_1STEP), (500, TOL_1000)):
        g, _ = run(er, w, n_steps)
        st, s, _, _ = orc.step(w, n_steps=n_steps)
        assert s == 0
        assert_parity(w, g, (st.positions, st.velocities, st.directors, st.omega), tol, raw=("r", "Q"),
                      label=f"warp kernel features x{n_steps}")


def test_warp_temporal_blocking_and_graphs(er, monkeypatch):
    """Several steps per launch (the tile kept in registers) and CUDA-graph step launches give the
    trajectory of one launch per step, bitwise."""
    w = uniform_batch(16, 2000, seed=3)
    a, _ = run(er, w, 96)                       # 3 graph launches of 32 steps
    b, _ = run(er, w, 96, spl=8)                # temporal blocking, 12 launches
    monkeypatch.setenv("ER_NO_STEP_GRAPH", "1")
    c, _ = run(er, w, 96)
    monkeypatch.delenv("ER_NO_STEP_GRAPH")
    same(a, b)
    same(a, c)


@pytest.mark.parametrize("nb", ["2", "3", "4"])
def test_warp_stage_buffers(er, monkeypatch, nb):
    """The pipeline depth (stage buffers per CTA) changes nothing but timing."""
    w = uniform_batch(16, 5000, seed=4)
    ref, _ = run(er, w, 20)
    monkeypatch.setenv("ER_WARP_BUFFERS", nb)
    out, _ = run(er, w, 20)
    monkeypatch.delenv("ER_WARP_BUFFERS")
    same(ref, out)


@pytest.mark.parametrize("N,R", [(16, 3000), (5, 700), (29, 300)])
def test_warp_stream_equals_tile_pipelined(er, monkeypatch, N, R):
    """The per-warp streaming pipeline (default) and the tile-pipelined warp kernel (ER_WARP_TMA=1)
    give the same trajectory bitwise, with actuation and static rest curvature too."""
    w = uniform_batch(N, R, seed=30 + N)
    rng = np.random.default_rng(N)
    w.act_A, w.act_f, w.act_L = rng.uniform(0.5, 2, R), rng.uniform(0.5, 2, R), np.full(R, 0.1)
    w.rest_kappa = rng.standard_normal((w.n_voronoi_total, 3)) * 0.5
    a, _ = run(er, w, 30)
    monkeypatch.setenv("ER_WARP_TMA", "1")
    b, _ = run(er, w, 30)
    monkeypatch.delenv("ER_WARP_TMA")
    same(a, b)


def test_warp_fault_reports_rod(er):
    w = uniform_batch(16, 100, seed=5)
    w.clamp[57] = 0                                 # node N free (a clamped node's v is reset)
    no = w.node_offsets()
    bad = w.velocities.copy()
    bad[no[57] + 16, 2] = np.nan                    # node N (the rod's last lane holds it)
    with er.RodBatch(w) as b:
        b.set_state(velocities=bad)
        with pytest.raises(er.ErError):
            b.step(2, w.dt)
        rod_id, bits = b.fault()
        assert rod_id == 57 and bits & er.ER_F_NONFINITE


def test_pair_features_equal_tile_kernel(er, monkeypatch):
    """Rods of 33..64 elements on warp pairs (mailbox exchanges across the two warps) with actuation,
    static rest curvature, per-element material, sigma0, magnetisation, muscle wave, external loads."""
    w = uniform_batch(50, 60, seed=71)
    rng = np.random.default_rng(72)
    R, E = w.n_rods, w.n_elems_total
    w.act_A, w.act_f, w.act_L = rng.uniform(0.5, 2, R), rng.uniform(0.5, 2, R), np.full(R, 0.1)
    w.rest_kappa = rng.standard_normal((w.n_voronoi_total, 3)) * 0.5
    same(run(er, w, 40)[0], run(er, w, 40, warp=False, monkeypatch=monkeypatch)[0])
    rod_of = np.repeat(np.arange(R), w.n_elems)
    for name in ("density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c"):
        setattr(w, name, getattr(w, name)[rod_of] * rng.uniform(0.9, 1.1, E))
    w.rest_sigma = rng.standard_normal((E, 3)) * 1e-4
    w.magnetization = rng.standard_normal((E, 3)) * 1e-4
    w.b_field, w.b_omega = np.array([1e-2, 0.0, 5e-3]), 30.0
    w.musc_A, w.musc_T = rng.uniform(1e-9, 1e-8, R), rng.uniform(0.5, 2, R)
    w.musc_lambda, w.musc_phi = rng.uniform(0.05, 0.1, R), rng.uniform(0, 6, R)
    w.ext_force = rng.standard_normal((w.n_nodes_total, 3)) * 1e-7
    w.ext_couple = rng.standard_normal((E, 3)) * 1e-10
    same(run(er, w, 40)[0], run(er, w, 40, warp=False, monkeypatch=monkeypatch)[0])


def test_pair_full_cfg4_sampled(er, orc):
    """BASELINE configs[3] (65,536 rods of 64 elements, actuation) at full size on warp pairs,
    1000 steps, 32 sampled rods re-run by the oracle."""
    w = W.make("cfg4")
    with er.RodBatch(w) as b:
        assert b.info().warp_rod_elems == 64
        b.step(1000, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    rods = W.sample_rods(w, 32, seed=13)
    ws = w.subset(rods)
    no, eo = w.node_offsets(), w.elem_offsets()
    nidx = np.concatenate([np.arange(no[r], no[r + 1]) for r in rods])
    eidx = np.concatenate([np.arange(eo[r], eo[r + 1]) for r in rods])
    st, s, _, _ = orc.step(ws, n_steps=1000)
    assert s == 0 and t == st.t
    assert_parity(ws, (pos[nidx], vel[nidx], dirs[eidx], om[eidx]), (st.positions, st.velocities, st.directors, st.omega),
                  TOL_1000, raw=("r", "Q"), label="cfg4 full x1000, warp pairs")


def test_warp_full_cfg3_sampled(er, orc):
    """BASELINE configs[2] at full size on the warp kernel (bench.py's configuration), 1000 steps,
    48 sampled rods re-run by the oracle."""
    w = W.make("cfg3")
    with er.RodBatch(w) as b:
        assert b.info().warp_rod_elems == 16
        b.step(1000, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    rods = W.sample_rods(w, 48, seed=11)
    ws = w.subset(rods)
    no, eo = w.node_offsets(), w.elem_offsets()
    nidx = np.concatenate([np.arange(no[r], no[r + 1]) for r in rods])
    eidx = np.concatenate([np.arange(eo[r], eo[r + 1]) for r in rods])
    st, s, _, _ = orc.step(ws, n_steps=1000)
    assert s == 0 and t == st.t
    assert_parity(ws, (pos[nidx], vel[nidx], dirs[eidx], om[eidx]), (st.positions, st.velocities, st.directors, st.omega),
                  TOL_1000, raw=("r", "Q"), label="cfg3 full x1000, warp kernel")


def test_contact_relayouts_warp_batch(er):
    """Contact runs the tile kernels: er_set_contact re-lays a warp-layout batch out into rod-aligned
    tiles; the state survives bitwise and the trajectory equals a batch created in the tile layout."""
    import os
    w = W.make("fibres").subset(np.arange(256))
    wnc = dataclasses.replace(w, contact=None)
    with er.RodBatch(wnc) as b:
        assert b.info().warp_rod_elems == 16
        b.step(3, w.dt)
        before = b.get_state()
        b.set_contact(w.contact)
        assert b.info().warp_rod_elems == 0
        after = b.get_state()
        same(before, after)
        b.step(20, w.dt)
        a = b.get_state()
    os.environ["ER_NO_WARP"] = "1"
    try:
        with er.RodBatch(wnc) as b:
            b.step(3, w.dt)
            b.set_contact(w.contact)
            b.step(20, w.dt)
            ref = b.get_state()
    finally:
        del os.environ["ER_NO_WARP"]
    same(a, ref)


def test_warp_faults_antipodal_degenerate_overspeed(er, orc):
    """The warp kernel's fault word: an adjacent relative rotation near pi, a collapsed element and an
    overspeeding node each report their rod (canonical id), like the tile kernel and the oracle."""
    import scipy.linalg as sla
    K = lambda v: np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])
    base = uniform_batch(16, 40, seed=91, clamp_mix=False, tip=False)
    base.velocities[:] = 0.0
    base.omega[:] = 0.0
    no, eo = base.node_offsets(), base.elem_offsets()
    # antipodal: rod 23, elements 9.. turned by pi - 1e-8 about an axis
    w = dataclasses.replace(base, directors=base.directors.copy())
    a = np.array([0.2, -0.5, 1.0]) / np.linalg.norm([0.2, -0.5, 1.0])
    w.directors[eo[23] + 9:eo[24]] = sla.expm((np.pi - 1e-8) * K(a)) @ w.directors[eo[23] + 8]  # relative turn = R
    with er.RodBatch(w) as b:
        assert b.info().warp_rod_elems == 16
        with pytest.raises(er.ErError):
            b.step(1, 1e-9)
        rod_id, bits = b.fault()
        assert rod_id == 23 and bits & er.ER_F_ANTIPODAL
    st, s, bad, bits = orc.step(w, n_steps=1, dt=1e-9)
    assert bad == 23 and bits & orc.F_ANTIPODAL
    # degenerate: rod 31's element 15 (the lane that also owns node N) collapses
    w = dataclasses.replace(base, positions=base.positions.copy())
    w.positions[no[31] + 16] = w.positions[no[31] + 15]
    with er.RodBatch(w) as b:
        with pytest.raises(er.ErError):
            b.step(1, 1e-9)
        rod_id, bits = b.fault()
        assert rod_id == 31 and bits & er.ER_F_DEGENERATE
    # overspeed on node N of rod 7
    w = dataclasses.replace(base, velocities=base.velocities.copy())
    w.velocities[no[7] + 16, 0] = 1e12
    with er.RodBatch(w) as b:
        with pytest.raises(er.ErError):
            b.step(1, 1e-12)
        rod_id, bits = b.fault()
        assert rod_id == 7 and bits & er.ER_F_OVERSPEED
