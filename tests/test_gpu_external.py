"""User external loads f and c-bar of Eqs. (1a)-(1b) (er_set_external_loads;
reading DESIGN §3 #30): parity against the oracle on packed ragged batches, long (cluster) rods and
contact batches; device-resident loads updated every step (the FSI coupling of PAPER.md:198);
step graphs pick up new values; clearing restores the load-free kernel bitwise."""
import dataclasses

import numpy as np
import pytest

import workloads as W
from parity import TOL_1000, TOL_1STEP, assert_parity
from test_gpu_long import perturbed
from test_gpu_parity import RAW, RAW_1000

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


def per_elem(w, a):
    a = np.asarray(a, float)
    return a if a.shape[0] == w.n_elems_total else np.repeat(a, w.n_elems)


def loads(w, seed, acc=5.0, alpha=50.0):
    """Random node forces of m_i * N(0, acc) and element couples of J * N(0, alpha): loads of
    the size of the gravity / inertial terms, in canonical order."""
    rng = np.random.default_rng(seed)
    rho, A = per_elem(w, w.density), per_elem(w, w.area)
    I1, I2 = per_elem(w, w.I1), per_elem(w, w.I2)
    me = rho * A * w.rest_lengths
    m = np.zeros(w.n_nodes_total)
    no, eo = w.node_offsets(), w.elem_offsets()
    for r in range(w.n_rods):
        s = me[eo[r]:eo[r + 1]]
        m[no[r]:no[r + 1] - 1] += s / 2
        m[no[r] + 1:no[r + 1]] += s / 2
    J = rho[:, None] * w.rest_lengths[:, None] * np.stack([I1, I2, I1 + I2], axis=1)
    return m[:, None] * rng.normal(0, acc, (w.n_nodes_total, 3)), J * rng.normal(0, alpha, (w.n_elems_total, 3))


def with_loads(w, seed, **kw):
    f, c = loads(w, seed, **kw)
    return dataclasses.replace(w, ext_force=f, ext_couple=c)


def run_gpu(er, w, n_steps):
    with er.RodBatch(w) as b:
        b.step(n_steps, w.dt)
        return b.get_state()[:4]


def run_orc(orc, w, n_steps, state=None):
    st, s, bad, bits = orc.step(w, state, n_steps=n_steps)
    assert s == 0, (bad, bits)
    return st


def tup(st):
    return st.positions, st.velocities, st.directors, st.omega


@pytest.mark.parametrize("name,n", [("cfg5", 150), ("cfg3", 300), ("cfg4", 64)])
def test_parity(er, orc, name, n):
    w = W.make(name, n_rods=n) if name != "cfg5" else W.make(name).subset(W.sample_rods(W.make(name), n, seed=3))
    w = with_loads(w, seed=1)
    assert_parity(w, run_gpu(er, w, 1), tup(run_orc(orc, w, 1)), TOL_1STEP, raw=RAW[name],
                  label=f"{name} loads 1 step")
    assert_parity(w, run_gpu(er, w, 1000), tup(run_orc(orc, w, 1000)), TOL_1000, raw=RAW_1000[name],
                  label=f"{name} loads 1000 steps")


def test_long_rods(er, orc):
    w = with_loads(perturbed([700, 9, 1300, 300], seed=5), seed=2)
    assert_parity(w, run_gpu(er, w, 1), tup(run_orc(orc, w, 1)), TOL_1STEP, raw=("r", "v", "Q"),
                  label="long rods loads 1 step")
    assert_parity(w, run_gpu(er, w, 200), tup(run_orc(orc, w, 200)), TOL_1000, raw=("r", "Q"),
                  label="long rods loads 200 steps")


def test_with_contact(er, orc):
    """Loads pressing the fibre stacks together (-z on every node) on top of contact."""
    w = W.make("fibres", n_rods=64)
    f, c = loads(w, seed=4, acc=20.0)
    f[:, 2] -= np.abs(f[:, 2])
    w = dataclasses.replace(w, ext_force=f, ext_couple=c)
    assert_parity(w, run_gpu(er, w, 1), tup(run_orc(orc, w, 1)), TOL_1STEP, raw=("r", "v", "Q"),
                  label="fibres loads 1 step")
    assert_parity(w, run_gpu(er, w, 300), tup(run_orc(orc, w, 300)), TOL_1000, raw=("r", "Q"),
                  label="fibres loads 300 steps")


def test_device_loads_updated_every_step(er, orc):
    """A solver loop: new loads every step from device tensors (no host round trip), equal
    bitwise to host-sourced loads and within parity of the oracle fed the same sequence."""
    import torch
    w = W.make("cfg5").subset(W.sample_rods(W.make("cfg5"), 60, seed=9))
    seq = [loads(w, seed=100 + n) for n in range(25)]
    outs = []
    for device in (True, False):
        with er.RodBatch(w) as b:
            for f, c in seq:
                if device:
                    b.set_external_loads(torch.from_numpy(f).cuda(), torch.from_numpy(c).cuda())
                else:
                    b.set_external_loads(f, c)
                b.step(1, w.dt)
            outs.append(b.get_state()[:4])
    for x, y in zip(*outs):
        assert np.array_equal(x, y)
    st = None
    for f, c in seq:
        st = run_orc(orc, dataclasses.replace(w, ext_force=f, ext_couple=c), 1, st)
    assert_parity(w, outs[0], tup(st), TOL_1000, raw=("r", "Q"), label="per-step loads")


def test_new_values_reach_step_graphs(er, orc):
    """Multi-step calls run through captured step graphs; new load values (same buffers) must
    be seen by the next call, and a cleared array must stop acting."""
    w = W.make("cfg4", n_rods=40)
    f1, c1 = loads(w, seed=7)
    f2, _ = loads(w, seed=8)
    with er.RodBatch(w) as b:
        b.set_external_loads(f1, c1)
        b.step(64, w.dt)
        b.set_external_loads(f2, c1)
        b.step(64, w.dt)
        b.set_external_loads(f2, None)
        b.step(64, w.dt)
        g = b.get_state()[:4]
    st = run_orc(orc, dataclasses.replace(w, ext_force=f1, ext_couple=c1), 64)
    st = run_orc(orc, dataclasses.replace(w, ext_force=f2, ext_couple=c1), 64, st)
    st = run_orc(orc, dataclasses.replace(w, ext_force=f2), 64, st)
    assert_parity(w, g, tup(st), TOL_1000, raw=("r", "Q"), label="graph reloads")


def test_clear_restores_load_free_path(er):
    w = W.make("cfg5").subset(W.sample_rods(W.make("cfg5"), 50, seed=4))
    ref = run_gpu(er, w, 30)
    f, c = loads(w, seed=5)
    with er.RodBatch(w) as b:
        b.set_external_loads(f, c)
        b.set_external_loads(None, None)
        b.step(30, w.dt)
        out = b.get_state()[:4]
    for x, y in zip(out, ref):
        assert np.array_equal(x, y)
    with er.RodBatch(w) as b:                 # zero loads: the loaded kernel, same arithmetic
        b.set_external_loads(np.zeros_like(f), np.zeros_like(c))
        b.step(30, w.dt)
        out = b.get_state()[:4]
    assert_parity(w, out, ref, 1e-14, raw=("r", "Q"), label="zero loads")
    with er.RodBatch(w) as b:
        with pytest.raises(ValueError):
            b.set_external_loads(f[:-1], None)


def test_distributed_load_cantilever_statics(er):
    """A cantilever under a uniform distributed force (node shares q lhat, ends q lhat/2) relaxes
    on the GPU (temporal blocking, 250,000 steps) to the beam-theory tip deflection
    q L^4/(8EI) + q L^2/(2 ac G A) at the clamp's effective length -- the oracle pin of
    tests/test_oracle_external.py, reached by the CUDA path."""
    from rodkit import rod
    N, L, q = 100, 1.0, 1e-3
    lh = L / N
    w = rod(N=N, L=L, r=0.01, clamp=0, nu=1.2, dt=1e-4)
    f = np.zeros((N + 1, 3))
    f[1:N, 0] = q * lh
    f[0, 0] = f[N, 0] = q * lh / 2
    w = dataclasses.replace(w, ext_force=f)
    with er.RodBatch(w) as b:
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, 1000)
        b.step(250000, w.dt)
        pos, vel, _, _, _ = b.get_state()
    assert np.max(np.abs(vel)) < 1e-5
    E, I, A, G, ac = w.youngs[0], w.I1[0], w.area[0], w.shear_mod[0], w.alpha_c[0]
    Le = L - lh / 2
    expect = q * Le ** 4 / (8 * E * I) + q * Le ** 2 / (2 * ac * G * A)
    assert abs(pos[-1, 0] / expect - 1) < 1e-3, pos[-1, 0] / expect - 1
