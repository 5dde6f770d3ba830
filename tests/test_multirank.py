"""Multi-rank host logic on CPU (gloo, world size 2): the rod sharding bench.py uses and the
scalar-diagnostics all-reduce (the only cross-GPU exchange).  The per-rank
compute here is the oracle (a CPU stand-in for the GPU shard); the point is the host logic:
every rod in exactly one shard, slot-balanced cuts, and all-reduced diagnostics equal to the
single-process ones."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import bench
import workloads as W


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_partition(world):
    w = W.make("cfg5", n_rods=997)
    shards = [bench.shard(w, r, world, "strong") for r in range(world)]
    assert sum(s.n_rods for s in shards) == w.n_rods
    assert np.array_equal(np.concatenate([s.n_elems for s in shards]), w.n_elems)
    slots = [int((s.n_elems + 1).sum()) for s in shards]
    assert max(slots) - min(slots) <= 2 * (int(w.n_elems.max()) + 1)
    assert np.array_equal(np.concatenate([s.positions for s in shards]), w.positions)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = W.make("cfg2", n_rods=10)
    ws = bench.shard(w, rank, world, "strong")
    st, s, _, _ = oracle.step(ws, n_steps=5)
    d = torch.tensor(oracle.energy(ws, st), dtype=torch.float64)
    vmax = d[9].clone()
    dist.all_reduce(d)
    dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
    d[9] = vmax
    if rank == 0:
        q.put(d.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_diagnostics_allreduce(orc):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.make("cfg2", n_rods=10)
    st, _, _, _ = orc.step(w, n_steps=5)
    ref = orc.energy(w, st)
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-300)
    assert got[9] == ref[9] and got[11] == ref[11]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_contact_shards_cut_between_stacks(world):
    """Contact workloads shard only at fibres-stack boundaries (stacks never touch), so every
    touching pair stays on one rank and no halo exchange is needed."""
    per = W.FIBRES["layers"] * W.FIBRES["per_layer"]
    w = W.make("fibres", n_rods=16 * per)
    shards = [bench.shard(w, r, world, "strong") for r in range(world)]
    assert sum(s.n_rods for s in shards) == w.n_rods
    assert all(s.n_rods % per == 0 for s in shards)
    assert np.array_equal(np.concatenate([s.positions for s in shards]), w.positions)


# ----------------------------------------------------------------------------- contact halo (CPU)
class _FakeBatch:
    """Stands in for RodBatch in the halo host logic: own node records are rank-tagged values."""

    def __init__(self, w, device=0, stream=None):
        self.n_nodes = w.n_nodes_total
        self.ghosts = None
        self.calls = []

    def set_contact_ghosts(self, *a):
        self.calls.append("ghosts")
        self.ghost_geom = a

    def set_contact(self, c):
        self.calls.append("contact")

    def step_begin(self, dt):
        self.calls.append("begin")

    def contact_records(self, out):
        out.copy_(self.own_records[: out.shape[0]])

    def set_ghost_records(self, src):
        self.ghosts = src.cpu().numpy().copy()

    def step_finish(self, dt):
        self.calls.append("finish")

    def close(self):
        pass


def _halo_worker(rank, world, port, q):
    import types

    import torch
    import torch.distributed as dist

    from paper_2605_13766_b200 import halo
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = W.make("fibres").subset(np.arange(48))
    cuts = [0, 17, 30, 48][: world + 1] if world == 3 else [0, 20, 48]
    fake = types.SimpleNamespace(RodBatch=_FakeBatch)
    sh = halo.ContactShard(fake, w, cuts, rank, world, device=0, batch_device="cpu")  # the fake lives on the CPU
    n = sh.nodes[rank]
    sh.batch.own_records = torch.full((n, 6), float(rank + 1), dtype=torch.float64) + \
        torch.arange(n, dtype=torch.float64)[:, None] * 1e-3
    sh.step(2, 1e-6)
    q.put((rank, sh.nodes, sh.batch.calls, sh.batch.ghosts, [np.asarray(x) for x in sh.batch.ghost_geom]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_contact_halo_exchange(world):
    """Every rank receives every other rank's node records, in rank order, each step (between
    er_step_begin and er_step_finish), and declares the other ranks' rods as ghosts."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((x[0], x[1:]) for x in (q.get(timeout=120) for _ in range(world)))
    for p in ps:
        p.join(timeout=60)
    w = W.make("fibres").subset(np.arange(48))
    cuts = [0, 17, 30, 48] if world == 3 else [0, 20, 48]
    for rank, (nodes, calls, ghosts, geom) in res.items():
        assert calls == ["ghosts", "contact", "begin", "finish", "begin", "finish"]
        expect = np.concatenate([np.full((nodes[k], 6), float(k + 1)) + np.arange(nodes[k])[:, None] * 1e-3
                                 for k in range(world) if k != rank])
        assert np.array_equal(ghosts, expect)
        others = np.concatenate([np.arange(cuts[k], cuts[k + 1]) for k in range(world) if k != rank])
        assert np.array_equal(geom[0], w.n_elems[others])
        assert geom[0].sum() + len(others) == sum(nodes[k] for k in range(world) if k != rank)
