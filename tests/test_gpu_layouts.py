"""Layout choices must not change results: the tile size (256-slot tiles with mid-length rods as
2-segment clusters vs 512-slot tiles), the packed rod order and temporal blocking give the same
trajectory bitwise, with every load type including user external loads; and the mid-length
cluster path is in parity with the oracle."""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import TOL_1000, TOL_1STEP, assert_parity
from rodkit import concat, rod
from test_gpu_external import loads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


def mixed_batch(n_short=1000, seed=7):
    """n_short rods of 20-60 elements plus rods of 256 and 300 elements (about 1.4% of the
    elements: the automatic rule takes 256-slot tiles and runs the two as 2-segment clusters),
    random orientations, perturbed directors, random rates, clamps, tip loads, gravity, damping."""
    rng = np.random.default_rng(seed)
    ns = list(rng.integers(20, 61, n_short)) + [256, 300]
    ws = []
    for q, N in enumerate(ns):
        Q0 = W.uniform_so3(rng, 1)[0]
        ws.append(rod(N=int(N), L=0.004 * N, r=0.002, E=1e6, Q=Q0, base=tuple(rng.uniform(-1, 1, 3)),
                      clamp=int(rng.integers(-1, 2)), nu=0.3, g=(0, 0, -9.81), dt=2e-6,
                      tip=tuple(rng.normal(0, 1e-6, 3))))
    w = concat(ws)
    w.tip_force = np.stack([x.tip_force[0] for x in ws])
    E = w.n_elems_total
    R = W.quat_to_rows(W.axis_angle_quat(rng.standard_normal((E, 3)), rng.uniform(0, 0.03, E)))
    w.directors = np.einsum("eab,ebc->eac", R, w.directors)
    w.velocities = rng.normal(0, 1e-3, w.velocities.shape)
    w.omega = rng.normal(0, 1e-2, w.omega.shape)
    return w


def run(er, w, n_steps, spl=1):
    with er.RodBatch(w) as b:
        if spl > 1:
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
        b.step(n_steps, w.dt)
        return b.get_state()[:4], b.info().tile_slots


def test_mid_length_clusters_match_512_tiles(er, orc, monkeypatch):
    w = mixed_batch()
    a, slots_a = run(er, w, 40)
    monkeypatch.setenv("ER_NO_MID_CLUSTERS", "1")
    b, slots_b = run(er, w, 40)
    assert (slots_a, slots_b) == (256, 512)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    monkeypatch.delenv("ER_NO_MID_CLUSTERS")
    st, s, _, _ = orc.step(w, n_steps=1)
    assert s == 0
    g, _ = run(er, w, 1)
    assert_parity(w, g, (st.positions, st.velocities, st.directors, st.omega), TOL_1STEP, raw=("r", "Q"),
                  label="mid-length clusters 1 step")
    st, s, _, _ = orc.step(w, n_steps=300)
    g, _ = run(er, w, 300)
    assert_parity(w, g, (st.positions, st.velocities, st.directors, st.omega), TOL_1000, raw=("r", "Q"),
                  label="mid-length clusters 300 steps")


def test_external_loads_invariant_to_layout(er, monkeypatch):
    """External loads (packed into the device order) with temporal blocking and without the
    packed rod order: the same trajectory bitwise."""
    w = mixed_batch(n_short=300, seed=3)
    f, c = loads(w, seed=9)
    w = dataclasses.replace(w, ext_force=f, ext_couple=c, act_A=np.full(w.n_rods, 0.5),
                            act_f=np.full(w.n_rods, 3.0), act_L=0.004 * w.n_elems.astype(float))
    ref, _ = run(er, w, 24)
    for out in (run(er, w, 24, spl=8)[0],):
        for x, y in zip(out, ref):
            assert np.array_equal(x, y)
    monkeypatch.setenv("ER_NO_PACK", "1")
    out, _ = run(er, w, 24)
    for x, y in zip(out, ref):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("case", ["one_tile", "two_tiles", "many_tiles", "ragged_long_loads"])
def test_sweeps_bitwise(er, case):
    """ER_OPT_SWEEPS_PER_LAUNCH: one launch streams all tiles S times (the reload of a CTA's first
    tile waits for its store: one, two and more tiles per CTA) -- bitwise the trajectory of one
    launch per step, also with long-rod clusters, external loads, actuation and on-chip steps."""
    if case == "one_tile":
        w = W.make("cfg2", n_rods=4)
    elif case == "two_tiles":
        w = W.make("cfg3", n_rods=6000)          # 400 tiles on 296 CTAs: one or two per CTA
    elif case == "many_tiles":
        w = W.make("cfg3", n_rods=15000)
    else:
        w = mixed_batch(n_short=800, seed=5)
        f, c = loads(w, seed=3)
        w = dataclasses.replace(w, ext_force=f, ext_couple=c, act_A=np.full(w.n_rods, 0.5),
                                act_f=np.full(w.n_rods, 3.0), act_L=0.004 * w.n_elems.astype(float))
    with er.RodBatch(w) as b:                   # one launch per step (CUDA-graph replays)
        b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, 1)
        b.step(37, w.dt)
        ref = b.get_state()[:4]
    for sweeps, spl in ((8, 1), (37, 1), (5, 3), (128, 1)):
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, sweeps)
            if spl > 1:
                b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
            b.step(37, w.dt)
            out = b.get_state()
        assert out[4] == b_t(w, 37)
        for x, y in zip(out[:4], ref):
            assert np.array_equal(x, y), (case, sweeps, spl)


def b_t(w, n):
    t = float(getattr(w, "t0", 0.0))
    for _ in range(n):
        th = t + 0.5 * w.dt
        t = th + 0.5 * w.dt
    return t


def test_while_graph_equals_chunked_graphs(er, monkeypatch):
    """The device-side WHILE step graph (one launch per er_step call) and its fallback (one graph
    launch per 32 steps) give the same trajectory bitwise, with long-rod clusters in the graph."""
    w = mixed_batch(n_short=300, seed=11)
    out = []
    for plain in (False, True):
        if plain:
            monkeypatch.setenv("ER_NO_WHILE_GRAPH", "1")
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, 1)
            b.step(100, w.dt)                       # 3 chunks of 32 + 4 plain launches
            b.step(64, w.dt)                        # 2 chunks
            out.append(b.get_state())
    for x, y in zip(out[0], out[1]):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_option_validation(er):
    w = W.make("cfg2", n_rods=4)
    with er.RodBatch(w) as b:
        for opt, bad in ((er.ER_OPT_SWEEPS_PER_LAUNCH, -1), (er.ER_OPT_STEPS_PER_LAUNCH, 0),
                         (er.ER_OPT_KERNEL, 9), (er.ER_OPT_PHASE_TIMING, 2), (99, 1)):
            with pytest.raises(er.ErError):
                b.set_option(opt, bad)
        b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, 0)   # automatic
        b.step(3, w.dt)
