"""Contact across GPUs (NEXT-4 with sharded rods): ghost rods and the split contact step.

- The split step (er_step_begin / er_step_finish) without ghosts is bitwise er_step.
- er_step refuses to run while ghosts are declared (their records would be stale).
- A `fibres` stack cut across two ranks (ranks sharing GPU 0 over gloo; paper_2605_13766_b200.halo
  exchanges the node records every step) follows the single-rank trajectory to round-off: the
  pair forces are evaluated from bit-identical inputs on both sides, only the order in which an
  element sums its partners' forces differs (parity gates of tests/parity.py).
"""
import dataclasses
import os

import numpy as np
import pytest

import bench
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


def stack():
    return W.make("fibres").subset(np.arange(W.FIBRES["layers"] * W.FIBRES["per_layer"]))


def test_split_step_equals_er_step(er):
    w = stack()
    with er.RodBatch(w) as b:
        b.step(25, w.dt)
        ref = b.get_state()
    with er.RodBatch(w) as b:
        for _ in range(25):
            b.step_begin(w.dt)
            b.step_finish(w.dt)
        out = b.get_state()
    for x, y in zip(ref, out):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_er_step_refused_with_ghosts(er):
    w = stack()
    with er.RodBatch(w) as b:
        b.set_contact_ghosts(np.array([4], np.int32), np.array([1e-3]), np.array([1.0]), np.array([0.01]),
                             np.array([0.01]))
        with pytest.raises(er.ErError) as ei:
            b.step(1, w.dt)
        assert "ghost" in str(ei.value)
        b.set_contact_ghosts(np.zeros(0, np.int32), np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0))
        b.step(1, w.dt)


def _rank(rank, world, port, cuts, n_steps, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2605_13766_b200 as er
    from paper_2605_13766_b200.halo import ContactShard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = stack()
    sh = ContactShard(er, w, cuts, rank, world, device=0)
    sh.step(n_steps, w.dt)
    pos, vel, dirs, om, t = sh.batch.get_state()
    st = sh.batch.contact_stats()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pos=pos, vel=vel, dirs=dirs, om=om, t=t,
             contacts=st.contacts)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_steps,tol", [(1, TOL_1STEP), (300, TOL_1000)])
def test_stack_cut_across_ranks_matches_one_rank(er, tmp_path, n_steps, tol):
    import torch.multiprocessing as mp
    w = stack()
    cuts = [0, w.n_rods // 2, w.n_rods]      # layers 0-7 | layers 8-15: crossings between layers 7 and 8
    mp.start_processes(_rank, args=(2, bench._free_port(), cuts, n_steps, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    with er.RodBatch(w) as b:
        b.step(n_steps, w.dt)
        full = b.get_state()
        contacts = b.contact_stats().contacts
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(2)]
    got = tuple(np.concatenate([p[k] for p in parts]) for k in ("pos", "vel", "dirs", "om"))
    assert all(float(p["t"]) == full[4] for p in parts)
    # every contact of the stack is seen by the rank(s) owning its elements: the cross-rank pairs by both
    assert sum(int(p["contacts"]) for p in parts) >= contacts
    assert_parity(w, got, full[:4], tol, raw=("r", "Q"), label=f"fibres stack over 2 ranks x{n_steps}")
