"""Contact across GPUs (SURVEY §8(f) NEXT-4 with rods sharded over ranks, §8(e)): host-side halo
exchange around the C-ABI's split contact step (include/er.h "contact across GPUs").

Each rank owns a contiguous shard of the rods in its RodBatch; the other ranks' rods enter as ghost
rods (contact geometry only).  Every step: er_step_begin (drift-1; own node records written on the
device) -> the node records of every rank are all-gathered over torch.distributed (NCCL device
tensors, or host tensors over gloo) -> the other ranks' records become this batch's ghost records ->
er_step_finish (contact over own + ghost elements, kick, drift-2).  Every rank sees every other
rank's rods, so the set of possible contacts is complete by construction (no spatial cut-off to
get wrong); the cost is one all-gather of 48 bytes per node per step.  Argument marshalling and
communication only: every step of the path runs in the library's kernels.
"""
from __future__ import annotations

import dataclasses

import numpy as np


def ghost_geometry(w, rods):
    """Contact geometry of `rods` (canonical ids of workload w) as ghost rods: elements per rod,
    contact radius (Contact.radius, else sqrt(A/pi) of the rod's first element), stiffness scale
    E r, shortest and longest rest element length."""
    rods = np.asarray(rods, dtype=np.int64)
    eo = w.elem_offsets()
    per_rod = w.density.shape[0] == w.n_rods
    first = eo[rods]
    area = w.area[rods] if per_rod else w.area[first]
    youngs = w.youngs[rods] if per_rod else w.youngs[first]
    c = getattr(w, "contact", None)
    radius = (np.asarray(c.radius, float)[rods] if c is not None and c.radius is not None
              else np.sqrt(area / np.pi))
    lmin = np.array([w.rest_lengths[eo[r]:eo[r + 1]].min() for r in rods])
    lmax = np.array([w.rest_lengths[eo[r]:eo[r + 1]].max() for r in rods])
    return dict(n_elems=w.n_elems[rods].astype(np.int32), radius=radius, stiffness=youngs * radius,
                lhat_min=lmin, lhat_max=lmax)


class ContactShard:
    """This rank's part of a contact workload `w` split into contiguous rod ranges `cuts`
    (cuts[k]..cuts[k+1] belong to rank k)."""

    def __init__(self, er, w, cuts, rank, world, device=0, stream=None, batch_device=None):
        """batch_device: where the batch's record buffers live (default the rank's GPU)."""
        import torch
        import torch.distributed as dist
        self.dist, self.torch = dist, torch
        self.rank, self.world, self.device = rank, world, device
        self.own = np.arange(cuts[rank], cuts[rank + 1])
        others = np.concatenate([np.arange(cuts[k], cuts[k + 1]) for k in range(world) if k != rank])
        c = w.contact
        w_own = w.subset(self.own)
        w_own = dataclasses.replace(w_own, contact=None)
        self.batch = er.RodBatch(w_own, device=device, stream=stream)
        g = ghost_geometry(w, others)
        self.batch.set_contact_ghosts(g["n_elems"], g["radius"], g["stiffness"], g["lhat_min"], g["lhat_max"])
        radius = None if c.radius is None else np.asarray(c.radius, float)[self.own]
        self.batch.set_contact(dataclasses.replace(c, radius=radius))
        nodes = [int(w.n_elems[cuts[k]:cuts[k + 1]].sum()) + (cuts[k + 1] - cuts[k]) for k in range(world)]
        self.nodes = nodes
        self.nmax = max(nodes)
        self.nccl = dist.get_backend() == "nccl"
        self.bdev = batch_device or f"cuda:{device}"
        dev = self.bdev if self.nccl else "cpu"
        self.send = torch.zeros((self.nmax, 6), dtype=torch.float64, device=dev)
        self.recv = [torch.zeros_like(self.send) for _ in range(world)]
        self.stage = torch.zeros((self.nmax, 6), dtype=torch.float64, device=self.bdev)

    def step(self, n_steps, dt):
        torch, dist = self.torch, self.dist
        own_n = self.nodes[self.rank]
        for _ in range(n_steps):
            self.batch.step_begin(dt)
            if self.nccl:
                self.batch.contact_records(self.send[:own_n])
            else:
                self.batch.contact_records(self.stage[:own_n])
                self.send[:own_n].copy_(self.stage[:own_n])
            dist.all_gather(self.recv, self.send)
            ghosts = torch.cat([self.recv[k][:self.nodes[k]] for k in range(self.world) if k != self.rank])
            if not self.nccl:
                ghosts = ghosts.to(self.bdev)
            self.batch.set_ghost_records(ghosts.contiguous())
            self.batch.step_finish(dt)

    def close(self):
        self.batch.close()
