"""Small run of every kernel path (for compute-sanitizer where it is available -- it is closed on
this GPU pool -- and as a plain all-paths smoke run):
tile kernels (fused, staged, one tile per CTA; temporal blocking; step graphs), long rods
(clusters, incl. 2-segment mid-length rods), contact, external loads (host and device)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import workloads as W
import paper_2605_13766_b200 as er
from rodkit import concat, rod

quick = "--quick" in sys.argv
for name, n in (("cfg2", 24), ("cfg5", 6), ("cfg4", 8)):
    w = W.make(name, n_rods=n)
    for kernel in ((0,) if quick else (0, 1, 2)):
        with er.RodBatch(w) as b:
            b.set_option(er.ER_OPT_KERNEL, kernel)
            b.step(3, w.dt)
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, 4)
            b.step(8, w.dt)
            b.diagnostics()
            b.get_state()
# step graphs (>= 32 launches per call)
w = W.make("cfg3", n_rods=64)
with er.RodBatch(w) as b:
    b.step(40, w.dt)
    b.get_state()
# long rods: a 600-element rod (3 segments), a 300-element rod beside short ones (2-segment
# cluster under the automatic tile rule), clamps and tip loads
rng = np.random.default_rng(1)
ws = [rod(N=600, L=1.2, r=0.004, clamp=0, tip=(0, 1e-5, 0), nu=0.1)]
ws += [rod(N=int(k), L=0.002 * int(k), r=0.002, base=(0.1 * q, 0, 0), tip=(0, 0, 0), nu=0.1)
       for q, k in enumerate(rng.integers(20, 60, 600))]
ws += [rod(N=300, L=0.6, r=0.004, base=(0, 1, 0), tip=(0, 0, 0), nu=0.1)]
wl = concat(ws)
for spl in (1, 3):
    with er.RodBatch(wl) as b:
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
        b.step(6, wl.dt)
        b.diagnostics()
        b.get_state()
# external loads, host then device
f = rng.normal(0, 1e-6, wl.positions.shape)
c = rng.normal(0, 1e-9, wl.omega.shape)
with er.RodBatch(wl) as b:
    b.set_external_loads(f, c)
    b.step(4, wl.dt)
    b.set_external_loads(torch.from_numpy(f).cuda(), torch.from_numpy(c).cuda())
    b.step(4, wl.dt)
    b.set_external_loads(None, None)
    b.step(2, wl.dt)
    b.get_state()
# contact
wc = W.make("fibres", n_rods=16)
for kernel in ((0,) if quick else (0, 1)):
    with er.RodBatch(wc) as b:
        b.set_option(er.ER_OPT_KERNEL, kernel)
        b.step(4, wc.dt)
        b.contact_stats()
        b.get_state()
print("sanitize run ok")
