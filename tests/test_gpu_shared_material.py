"""Shared-material batches on the warp kernels (DESIGN §4 "Shared material").

When every rod of a warp-layout batch has the same material constants (cfg3, cfg4: one filament
type), the 17 shared constants travel in the kernel parameters and each rod streams a 48-byte record
(tip force, actuation, flags) instead of the 192-byte one.  The arithmetic is the same, so the
trajectory must be bitwise that of the full-record kernel (ER_NO_UNI=1) and of the tile kernel
(ER_NO_WARP=1), and the library must fall back to full records as soon as a forcing change makes
the rods differ (per-rod damping), and return when they agree again (a captured step graph must
not keep stale constants).
"""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import TOL_1000, TOL_1STEP, assert_parity
from test_gpu_warp import er, force_warp_layout, same, uniform_batch  # noqa: F401  (fixtures)

pytestmark = pytest.mark.gpu


def shared_batch(N, R, seed, act=False, kappa0=False):
    """uniform_batch's rods (clamps at either end or free, tip loads, random frames) with one material
    and one damping rate for all rods."""
    w = uniform_batch(N, R, seed)
    rng = np.random.default_rng(seed + 1)
    w = dataclasses.replace(w, **W._rod_material(R, 1e-3, 2e6), damping=np.full(R, 0.1))
    if act:
        w.act_A, w.act_f, w.act_L = rng.uniform(0.5, 2, R), rng.uniform(0.5, 2, R), np.full(R, 0.1)
        w.act_component = 0
    if kappa0:
        w.rest_kappa = rng.standard_normal((w.n_voronoi_total, 3)) * 0.5
    return w


def run(er, w, n_steps, monkeypatch, env=None, forcing_seq=()):
    """n_steps steps, then for each (forcing kwargs, steps) of forcing_seq: set_forcing + steps.
    Returns the state and the shared_material flag seen before each stepping phase."""
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    try:
        with er.RodBatch(w) as b:
            flags = [b.info().shared_material]
            b.step(n_steps, w.dt)
            for kw, n in forcing_seq:
                b.set_forcing(**kw)
                flags.append(b.info().shared_material)
                b.step(n, w.dt)
            out = b.get_state()
    finally:
        for k in (env or {}):
            monkeypatch.delenv(k)
    return out, flags


@pytest.mark.parametrize("N,R,act,kappa0", [(16, 700, False, False), (16, 301, True, True), (7, 333, True, False),
                                            (4, 301, True, False), (32, 90, False, True), (33, 41, True, True),
                                            (64, 70, True, False), (45, 60, False, False)])
def test_shared_material_bitwise(er, monkeypatch, N, R, act, kappa0):
    w = shared_batch(N, R, seed=300 + N, act=act, kappa0=kappa0)
    a, fa = run(er, w, 64, monkeypatch)
    b, fb = run(er, w, 64, monkeypatch, env={"ER_NO_UNI": "1"})
    c, fc = run(er, w, 64, monkeypatch, env={"ER_NO_WARP": "1"})
    assert fa == [1] and fb == [0] and fc == [0]
    same(a, b)
    same(a, c)


def test_shared_material_parity(er, orc, monkeypatch):
    w = shared_batch(16, 200, seed=41, act=True)
    for n_steps, tol in ((1, TOL_1STEP), (1000, TOL_1000)):
        g, f = run(er, w, n_steps, monkeypatch)
        assert f == [1]
        st, s, _, _ = orc.step(w, n_steps=n_steps)
        assert s == 0
        assert_parity(w, g, (st.positions, st.velocities, st.directors, st.omega), tol, raw=("r", "Q"),
                      label=f"shared material x{n_steps}")


def test_shared_material_follows_forcing(er, monkeypatch):
    """Uniform damping -> per-rod damping (full records) -> another uniform damping and gravity (shared
    constants re-read; 64-step runs go through captured step graphs)."""
    w = shared_batch(16, 3000, seed=5)
    R = w.n_rods
    rng = np.random.default_rng(6)
    seq = [(dict(gravity=(0, 0, -9.81), damping=rng.uniform(0.0, 0.3, R), tip_force=w.tip_force), 64),
           (dict(gravity=(0, 1.0, -9.81), damping_all=0.25, tip_force=w.tip_force), 64),
           (dict(gravity=(0, 1.0, -9.81), damping=np.full(R, 0.05)), 64)]
    a, fa = run(er, w, 64, monkeypatch, forcing_seq=seq)
    b, fb = run(er, w, 64, monkeypatch, env={"ER_NO_UNI": "1"}, forcing_seq=seq)
    assert fa == [1, 0, 1, 1] and fb == [0, 0, 0, 0]
    same(a, b)


def test_baseline_workloads_are_shared(er):
    """cfg3 and cfg4 (one filament type each) run the shared-material kernels."""
    for name in ("cfg3", "cfg4"):
        w = W.make(name, n_rods=4096)
        with er.RodBatch(w) as b:
            info = b.info()
            assert info.warp_rod_elems > 0 and info.shared_material == 1, (name, info.warp_rod_elems)


def test_pair_walk_direction_bitwise(er, monkeypatch):
    """pair_bulk walks the tiles in alternating directions across step-graph launches (L2 reuse); the
    trajectory equals plain launches in one direction bitwise."""
    w = shared_batch(64, 300, seed=77, act=True)
    a, fa = run(er, w, 96, monkeypatch)                                   # 3 graph chunks of 32 launches
    b, fb = run(er, w, 96, monkeypatch, env={"ER_NO_STEP_GRAPH": "1"})   # plain launches
    assert fa == fb == [1]
    same(a, b)
