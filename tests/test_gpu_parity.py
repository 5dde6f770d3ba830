"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Metric and tolerances: tests/parity.py (north_star: 1e-12 after one step,
1e-8 after 1000 steps).  Small cases span several tiles with a ragged tail; full-size cases
run in bench.py's launch configuration and compare sampled rods (rods are independent, so
the oracle can run any subset).
"""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import assert_directors_round_trip, TOL_1000, TOL_1STEP, assert_parity
from rodkit import concat, rod

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


def run_gpu(er, w, n_steps, steps_per_launch=1, kernel=0, dt=None):
    with er.RodBatch(w) as b:
        if steps_per_launch != 1:
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, steps_per_launch)
        if kernel:
            b.set_option(er.ER_OPT_KERNEL, kernel)
        b.step(n_steps, w.dt if dt is None else dt)
        pos, vel, dirs, om, t = b.get_state()
    return (pos, vel, dirs, om), t


def run_orc(orc, w, n_steps):
    st, s, bad, bits = orc.step(w, n_steps=n_steps)
    assert s == 0, (bad, bits)
    return (st.positions, st.velocities, st.directors, st.omega), st.t


RAW = {"cfg1": ("r", "Q"), "cfg2": ("r", "v", "Q", "w"), "cfg3": ("r", "Q"), "cfg4": ("r", "Q", "w"),
       "cfg5": ("r", "Q", "w")}
# After 1000 steps the raw ratio of the rates is bounded by the problem's own conditioning:
# the oracle perturbed by half an ulp moves raw v/w by > 1e-8 on cfg3 and cfg4
# (tests/test_conditioning.py), so raw is gated on r and Q only there; cfg5 is well conditioned
# (< 1e-9) and gated raw on all four; the floored metric (C.6) gates all four everywhere.
RAW_1000 = {"cfg1": ("r", "Q"), "cfg2": ("r", "v", "Q", "w"), "cfg3": ("r", "Q"), "cfg4": ("r", "Q"),
            "cfg5": ("r", "v", "Q", "w")}
SMALL = {"cfg1": None, "cfg2": 200, "cfg3": 600, "cfg4": 96, "cfg5": 120}


def small(name):
    n = SMALL[name]
    w = W.make(name)
    if n is None:
        return w
    return w.subset(np.arange(n)) if name in ("cfg3",) else w.subset(W.sample_rods(w, n, seed=1)) \
        if name == "cfg5" else W.make(name, n_rods=n)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_parity_one_step(er, orc, name):
    w = small(name)
    g, tg = run_gpu(er, w, 1)
    o, to = run_orc(orc, w, 1)
    assert tg == to
    assert_parity(w, g, o, TOL_1STEP, raw=RAW[name], label=f"{name} 1 step")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_parity_1000_steps(er, orc, name):
    w = small(name)
    if name == "cfg2":
        w = w.subset(np.arange(48))
    g, tg = run_gpu(er, w, 1000)
    o, to = run_orc(orc, w, 1000)
    assert tg == to
    assert_parity(w, g, o, TOL_1000, raw=RAW_1000[name], label=f"{name} 1000 steps")


def test_cfg1_full_run(er, orc):
    """cfg1 as configured (20000 steps); report-level tolerance (C.6)."""
    w = W.make("cfg1")
    g, _ = run_gpu(er, w, w.n_steps)
    o, _ = run_orc(orc, w, w.n_steps)
    assert_parity(w, g, o, 1e-7, label="cfg1 20000 steps")


@pytest.mark.parametrize("name,n_steps", [("cfg3", 1), ("cfg3", 1000), ("cfg5", 1), ("cfg5", 1000), ("cfg4", 1), ("cfg4", 1000), ("cfg2", 1000)])
def test_full_size_sampled(er, orc, name, n_steps):
    """Full BASELINE size on the GPU, in bench.py's launch configuration; the oracle re-runs
    a seeded sample of rods (first, last and random ones) and we compare those rods."""
    w = W.make(name)
    with er.RodBatch(w) as b:
        b.step(n_steps, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    rods = W.sample_rods(w, 48, seed=2)
    ws = w.subset(rods)
    no, eo = w.node_offsets(), w.elem_offsets()
    nidx = np.concatenate([np.arange(no[r], no[r + 1]) for r in rods])
    eidx = np.concatenate([np.arange(eo[r], eo[r + 1]) for r in rods])
    o, to = run_orc(orc, ws, n_steps)
    assert t == to
    tol = TOL_1STEP if n_steps == 1 else TOL_1000
    assert_parity(ws, (pos[nidx], vel[nidx], dirs[eidx], om[eidx]), o, tol,
                  raw=RAW[name] if n_steps == 1 else RAW_1000[name],
                  label=f"{name} full x {n_steps}")


def test_temporal_blocking_bitwise(er):
    w = W.make("cfg2", n_rods=64)
    a, ta = run_gpu(er, w, 200)
    b, tb = run_gpu(er, w, 200, steps_per_launch=16)
    assert ta == tb
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_staged_kernel_matches_fused(er):
    w = W.make("cfg4", n_rods=40)
    a, _ = run_gpu(er, w, 50)
    b, _ = run_gpu(er, w, 50, kernel=1)
    for x, y in zip(a, b):
        assert np.max(np.abs(x - y)) <= 1e-14 * max(1.0, np.max(np.abs(x)))


def test_deterministic(er):
    w = W.make("cfg5", n_rods=50)
    a, _ = run_gpu(er, w, 20)
    b, _ = run_gpu(er, w, 20)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_shard_equivalence(er):
    """Rods are independent: sharding a batch (different tile packing) is bitwise neutral."""
    w = W.make("cfg5", n_rods=60)
    full, _ = run_gpu(er, w, 30)
    A, B = w.subset(np.arange(23)), w.subset(np.arange(23, 60))
    a, _ = run_gpu(er, A, 30)
    b, _ = run_gpu(er, B, 30)
    for x, y, z in zip(full, a, b):
        assert np.array_equal(x, np.concatenate([y, z]))


def test_round_trip_host_and_device(er):
    import torch
    w = W.make("cfg5", n_rods=30)
    with er.RodBatch(w) as b:
        pos, vel, dirs, om, t = b.get_state()
        assert np.array_equal(pos, w.positions)
        assert_directors_round_trip(dirs, w.directors)
        assert np.array_equal(vel, w.velocities) and np.array_equal(om, w.omega) and t == 0.0
        dp = torch.empty((w.n_nodes_total, 3), dtype=torch.float64, device="cuda")
        dd = torch.empty((w.n_elems_total, 3, 3), dtype=torch.float64, device="cuda")
        b.get_state_into(positions=dp, directors=dd)
        assert np.array_equal(dp.cpu().numpy(), w.positions) and np.array_equal(dd.cpu().numpy(), dirs)
    wd = dataclasses.replace(w, positions=torch.tensor(w.positions, device="cuda"),
                             velocities=torch.tensor(w.velocities, device="cuda"),
                             directors=torch.tensor(w.directors, device="cuda"),
                             omega=torch.tensor(w.omega, device="cuda"))
    with er.RodBatch(wd) as b:
        pos, vel, dirs2, om, _ = b.get_state()
        assert np.array_equal(pos, w.positions) and np.array_equal(dirs2, dirs)


def test_diagnostics_match_oracle(er, orc):
    for name, n in (("cfg2", 30), ("cfg4", 20), ("cfg5", 25)):
        w = W.make(name, n_rods=n)
        with er.RodBatch(w) as b:
            b.step(10, w.dt)
            d = b.diagnostics()
        st, _, _, _ = orc.step(w, n_steps=10)
        ref = orc.energy(w, st)
        # sums with cancellation (gravity PE over rods on both sides of the origin, momentum):
        # tolerance relative to the magnitude of the summed terms, not of the sum
        mass, vmax = ref[10], ref[9]
        rmax = np.max(np.abs(st.positions))
        scale = max(np.max(np.abs(ref[:6])), mass * np.linalg.norm(w.gravity) * rmax)
        assert np.all(np.abs(d[:6] - ref[:6]) <= 1e-10 * np.abs(ref[:6]) + 1e-12 * scale), (name, d, ref)
        assert np.all(np.abs(d[6:9] - ref[6:9]) <= 1e-12 * mass * vmax), (name, d, ref)
        assert np.isclose(d[9], ref[9], rtol=1e-12) and np.isclose(d[10], ref[10], rtol=1e-13) and d[11] == ref[11]


# ----------------------------------------------------------------------------- edge cases
def test_empty_batch(er):
    w = W.make("cfg2", n_rods=1).subset(np.arange(0))
    with er.RodBatch(w) as b:
        b.step(10, 1e-5)
        pos, vel, dirs, om, t = b.get_state()
        assert pos.shape == (0, 3) and dirs.shape == (0, 3, 3)
        assert np.all(b.diagnostics()[:9] == 0)


def edge_batch():
    """N = 1, 2, 3 and a 511-element rod (the maximum), clamps at either end, tip loads on
    free and end-clamped rods, random perturbations so every term is active."""
    rng = np.random.default_rng(5)
    import scipy.linalg as sla

    def sk(v):
        return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])
    parts = []
    for N, cl, tip in ((1, -1, None), (2, 0, (1e-3, 0, 0)), (3, 1, (0, 1e-3, 1e-3)), (7, -1, (1e-4, 1e-4, 0)),
                       (511, 0, (0, 0, -1e-3)), (40, 1, None)):
        Q0 = sla.expm(sk(rng.standard_normal(3)))
        w = rod(N=N, L=0.01 * N, r=0.002, E=1e6, Q=Q0, clamp=cl, tip=tip if tip else (0, 0, 0), nu=0.3,
                g=(0, 0, -9.81), dt=1e-6)
        E = w.n_elems_total
        w.directors = np.stack([sla.expm(sk(rng.standard_normal(3) * 0.01)) for _ in range(E)]) @ w.directors
        w.velocities = rng.standard_normal(w.positions.shape) * 1e-3
        w.omega = rng.standard_normal((E, 3)) * 0.1
        parts.append(w)
    return concat(parts)


def test_edge_cases_parity(er, orc):
    w = edge_batch()
    for n in (1, 200):
        g, _ = run_gpu(er, w, n)
        o, _ = run_orc(orc, w, n)
        assert_parity(w, g, o, TOL_1STEP if n == 1 else TOL_1000, raw=("r", "v", "Q", "w"), label=f"edge x{n}")


def test_general_rods_parity(er, orc):
    """Non-uniform rest lengths and per-element material (the 'general' per-slot path)."""
    w = edge_batch().subset(np.array([1, 2, 3, 5]))
    rng = np.random.default_rng(8)
    E = w.n_elems_total
    w.rest_lengths = w.rest_lengths * rng.uniform(0.9, 1.1, E)
    eo = w.elem_offsets()
    rod_of = np.repeat(np.arange(w.n_rods), w.n_elems)
    for name in ("density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c"):
        setattr(w, name, getattr(w, name)[rod_of] * rng.uniform(0.8, 1.2, E))
    w.rest_sigma = rng.standard_normal((E, 3)) * 1e-3
    w.rest_kappa = rng.standard_normal((w.n_voronoi_total, 3)) * 0.5
    w.act_A, w.act_f, w.act_L = rng.uniform(0.5, 2, 4), rng.uniform(0.5, 2, 4), np.full(4, 0.3)
    w.act_component = 2
    w.magnetization = rng.standard_normal((E, 3)) * 1e-3
    w.b_field, w.b_omega = np.array([1e-2, 0.0, 5e-3]), 30.0
    w.b_axis = np.array([0.3, 1.0, -0.2])
    w.musc_A, w.musc_T = rng.uniform(1e-6, 1e-5, 4), rng.uniform(0.5, 2, 4)
    w.musc_lambda, w.musc_phi = rng.uniform(0.1, 0.5, 4), rng.uniform(0, 6, 4)
    w.musc_component = 1
    for n in (1, 200):
        g, _ = run_gpu(er, w, n)
        o, _ = run_orc(orc, w, n)
        assert_parity(w, g, o, TOL_1STEP if n == 1 else TOL_1000, raw=("r", "v", "Q", "w"), label=f"general x{n}")


def test_muscle_wave_parity(er, orc):
    """NEXT-3 muscular torque wave on uniform rods (couple pairs folded into the exchanged moment)."""
    w = W.make("cfg4", n_rods=24)
    R = w.n_rods
    rng = np.random.default_rng(12)
    w.act_A = w.act_f = w.act_L = None
    w.musc_A, w.musc_T = rng.uniform(1e-5, 1e-4, R), rng.uniform(0.5, 2, R)
    w.musc_lambda, w.musc_phi = rng.uniform(0.2, 1.0, R), rng.uniform(0, 6, R)
    for n in (1, 1000):
        g, _ = run_gpu(er, w, n)
        o, _ = run_orc(orc, w, n)
        assert_parity(w, g, o, TOL_1STEP if n == 1 else TOL_1000, raw=("r", "Q"), label=f"muscle x{n}")


def test_fault_reports_rod(er):
    """Fault injection: a NaN is rejected at create (validation) but injected with
    er_set_state it surfaces at the next er_step with the rod id."""
    w = W.make("cfg2", n_rods=20)
    no = w.node_offsets()
    bad = w.velocities.copy()
    bad[no[13] + 4, 1] = np.nan
    with pytest.raises(er.ErError):
        er.RodBatch(dataclasses.replace(w, velocities=bad))
    with er.RodBatch(w) as b:
        b.set_state(velocities=bad)
        with pytest.raises(er.ErError) as ei:
            b.step(3, w.dt)
        assert ei.value.status == er.ER_EUNSTABLE
        rod_id, bits = b.fault()
        assert rod_id == 13 and bits & er.ER_F_NONFINITE


def test_packed_rod_order(er, monkeypatch):
    """Ragged batches are stored in a best-fit-decreasing tile order (fewer, fuller tiles); the
    API stays canonical: the same trajectory bitwise as the identity order, forcing / clamps /
    fault ids in canonical rod numbering."""
    w = W.make("cfg5", n_rods=300)
    tip = np.zeros((w.n_rods, 3))
    tip[::7, 0] = 1e-4                                       # per-rod forcing in canonical order
    w = dataclasses.replace(w, tip_force=tip)
    out, tiles = [], []
    for pack in (True, False):
        if not pack:
            monkeypatch.setenv("ER_NO_PACK", "1")
        with er.RodBatch(w) as b:
            tiles.append(b.info().n_tiles)
            b.step(20, w.dt)
            out.append(b.get_state())
    assert tiles[0] < tiles[1]
    for x, y in zip(out[0], out[1]):
        assert np.array_equal(x, y)
    monkeypatch.delenv("ER_NO_PACK")
    no = w.node_offsets()
    bad = w.velocities.copy()
    for r in (250, 77):
        bad[no[r] + 2, 0] = np.inf
    with er.RodBatch(w) as b:
        b.set_state(velocities=bad)
        with pytest.raises(er.ErError):
            b.step(2, w.dt)
        assert b.fault()[0] == 77


def test_fault_degenerate_and_overspeed(er, orc):
    w = concat([rod(N=4, L=0.2), rod(N=4, L=0.2), rod(N=4, L=0.2)])
    w.positions[11] = w.positions[10]
    w.positions[12:] = w.positions[10] + (w.positions[12:] - w.positions[11])
    with er.RodBatch(w) as b:
        with pytest.raises(er.ErError):
            b.step(1, 1e-9)
        assert b.fault()[0] == 2 and b.fault()[1] & er.ER_F_DEGENERATE
    st, s, bad, bits = orc.step(w, n_steps=1, dt=1e-9)
    assert bad == 2 and bits & orc.F_DEGENERATE
    w = concat([rod(N=4, L=0.2), rod(N=4, L=0.2)])
    w.velocities[7, 0] = 1e12
    with er.RodBatch(w) as b:
        with pytest.raises(er.ErError):
            b.step(1, 1e-12)
        assert b.fault()[0] == 1 and b.fault()[1] & er.ER_F_OVERSPEED


def test_pinned_host_zero_copy_paths(er):
    """Page-locked host arrays take the zero-copy layout path (the kernels read / write host
    memory over PCIe); pageable ones the staged copy.  Both give identical states, and the
    validation still runs on the zero-copy upload."""
    import torch
    w = W.make("cfg5", n_rods=40)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    tp = {k: pin(getattr(w, k)) for k in ("positions", "velocities", "directors", "omega")}
    wp = dataclasses.replace(w, **{k: v.numpy() for k, v in tp.items()})
    outs = [torch.empty_like(tp[k]).pin_memory() for k in ("positions", "velocities", "directors", "omega")]
    with er.RodBatch(wp) as b:
        b.step(7, w.dt)
        b.get_state_into(*[o.numpy() for o in outs])
    with er.RodBatch(w) as b:
        b.step(7, w.dt)
        ref = b.get_state()[:4]
    for o, r in zip(outs, ref):
        assert np.array_equal(o.numpy(), r)
    bad = tp["directors"].clone().pin_memory()
    bad[3] *= 1.01
    with pytest.raises(er.ErError) as ei:
        er.RodBatch(dataclasses.replace(wp, directors=bad.numpy()))
    assert "orthonormal" in str(ei.value)


def test_validation_collects_all_errors(er):
    w = W.make("cfg2", n_rods=4)
    w.directors[3] *= 1.01
    w.youngs[2] = -1.0
    with pytest.raises(er.ErError) as ei:
        er.RodBatch(w)
    msg = str(ei.value)
    assert "youngs" in msg and ei.value.status == er.ER_EINVAL
    w = W.make("cfg2", n_rods=4)
    w.directors[3] *= 1.01
    with pytest.raises(er.ErError) as ei:
        er.RodBatch(w)
    assert "orthonormal" in str(ei.value)


def test_set_state_resume_bitwise(er):
    w = W.make("cfg2", n_rods=12)
    full, _ = run_gpu(er, w, 30)
    with er.RodBatch(w) as b:
        b.step(10, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    with er.RodBatch(w) as b2:
        b2.set_state(pos, vel, dirs, om, t=t)
        b2.step(20, w.dt)
        rest = b2.get_state()[:4]
    for x, y in zip(full, rest):
        assert np.array_equal(x, y)


def test_resume_from_snapshot_bitwise(er):
    """Checkpoint/resume: get_state (incl. t) -> new batch -> same trajectory bitwise."""
    w = W.make("cfg4", n_rods=10)
    full, _ = run_gpu(er, w, 40)
    with er.RodBatch(w) as b:
        b.step(15, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    w2 = dataclasses.replace(w, positions=pos, velocities=vel, directors=dirs, omega=om, t0=t)
    rest, _ = run_gpu(er, w2, 25)
    for x, y in zip(full, rest):
        assert np.array_equal(x, y)


# ----------------------------------------------------------------------------- NEXT-2 cilia
@pytest.mark.parametrize("n_steps,tol", [(1, TOL_1STEP), (1000, TOL_1000)])
def test_cilia_carpet_parity(er, orc, n_steps, tol):
    w = W.make("cilia8")
    g, tg = run_gpu(er, w, n_steps)
    o, to = run_orc(orc, w, n_steps)
    assert tg == to
    assert_parity(w, g, o, tol, raw=("r", "Q"), label=f"cilia8 x{n_steps}")


def test_cilia_farm_sampled(er, orc):
    """111,797 magnetic cilia on the GPU; a seeded sample re-run by the oracle."""
    w = W.make("ciliafarm")
    with er.RodBatch(w) as b:
        b.step(200, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    rods = W.sample_rods(w, 32, seed=5)
    ws = w.subset(rods)
    no, eo = w.node_offsets(), w.elem_offsets()
    nidx = np.concatenate([np.arange(no[r], no[r + 1]) for r in rods])
    eidx = np.concatenate([np.arange(eo[r], eo[r + 1]) for r in rods])
    o, to = run_orc(orc, ws, 200)
    assert t == to
    assert_parity(ws, (pos[nidx], vel[nidx], dirs[eidx], om[eidx]), o, TOL_1000, raw=("r", "Q"), label="farm")


def test_step_graph_bitwise(er, monkeypatch):
    """Runs of >= 32 launches go through a CUDA graph (time carried on the device): bitwise the
    same as plain launches, for tile rods, ragged rods, long rods and temporal blocking."""
    w = W.make("cfg5", n_rods=40)
    out = []
    for plain in (False, True):
        if plain:
            monkeypatch.setenv("ER_NO_STEP_GRAPH", "1")
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, 1)      # one launch per step (graphs)
            b.step(70, w.dt)                                  # 2 graph launches + 6 plain steps
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, 3)
            b.step(100, w.dt)                                 # 1 graph launch (96 steps) + 4
            out.append(b.get_state())
    for x, y in zip(out[0], out[1]):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_fault_antipodal(er, orc):
    """Adjacent elements rotated by nearly pi against each other (SPEC.md:113 reading, ER_F_ANTIPODAL):
    the kernel flags the rod id; a rotation safely below the threshold is not flagged; the oracle
    agrees in both cases."""
    import scipy.linalg as sla
    K = lambda v: np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])
    for angle, flagged in ((np.pi - 1e-8, True), (np.pi - 1e-4, False)):
        parts = [rod(N=5, L=0.05, r=0.002) for _ in range(3)]
        a = np.array([0.3, 1.0, -0.4])
        a /= np.linalg.norm(a)
        R = sla.expm(angle * K(a))
        w = concat(parts)
        eo = w.elem_offsets()
        w.directors[eo[2] + 3:eo[3]] = R @ w.directors[eo[2] + 3]   # rod 2: elements 3.. turned by R
        with er.RodBatch(w) as b:
            if flagged:
                with pytest.raises(er.ErError) as ei:
                    b.step(1, 1e-9)
                assert ei.value.status == er.ER_EUNSTABLE
                rod_id, bits = b.fault()
                assert rod_id == 2 and bits & er.ER_F_ANTIPODAL, (rod_id, bits)
            else:
                b.step(1, 1e-9)
                assert b.fault()[1] & er.ER_F_ANTIPODAL == 0
        st, s, bad, bits = orc.step(w, n_steps=1, dt=1e-9)
        assert (bad == 2 and bits & orc.F_ANTIPODAL) if flagged else not (bits & orc.F_ANTIPODAL)


def test_step_graph_follows_dt_change(er, monkeypatch):
    """er_step may change dt between calls: the captured step graph holds the step size by value, so
    a call with a new dt must recapture it.  A batch large enough for one launch per
    step (no sweeps) and runs of >= 32 launches take the graph path; the result must equal plain
    launches bitwise and the oracle within the 1000-step gate."""
    w = W.make("cfg3").subset(np.arange(148 * 2 * 16 * 5))     # > 4 tiles per CTA: no sweeps
    out = []
    for plain in (False, True):
        if plain:
            monkeypatch.setenv("ER_NO_STEP_GRAPH", "1")
        with er.RodBatch(w) as b:
            b.step(64, w.dt)
            b.step(64, w.dt / 2)
            b.step(64, w.dt * 3)
            out.append(b.get_state())
    for x, y in zip(out[0], out[1]):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_temporal_blocking_full_size_vs_oracle(er, orc):
    """bench.py's temporal-blocking configuration (full cfg3, 100 steps per launch) against the
    oracle on sampled rods after 1000 steps (it was only checked transitively)."""
    w = W.make("cfg3")
    with er.RodBatch(w) as b:
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, 100)
        b.step(1000, w.dt)
        pos, vel, dirs, om, t = b.get_state()
    rods = W.sample_rods(w, 48, seed=7)
    ws = w.subset(rods)
    no, eo = w.node_offsets(), w.elem_offsets()
    nidx = np.concatenate([np.arange(no[r], no[r + 1]) for r in rods])
    eidx = np.concatenate([np.arange(eo[r], eo[r + 1]) for r in rods])
    o, to = run_orc(orc, ws, 1000)
    assert t == to
    assert_parity(ws, (pos[nidx], vel[nidx], dirs[eidx], om[eidx]), o, TOL_1000, raw=RAW_1000["cfg3"],
                  label="cfg3 full x 1000, 100 steps per launch")
