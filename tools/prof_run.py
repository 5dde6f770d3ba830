"""Small driver for ncu captures: one config, a few launches of the step kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2605_13766_b200 as er
name = sys.argv[1]; spl = int(sys.argv[2]); launches = int(sys.argv[3]); tile = int(sys.argv[4]) if len(sys.argv) > 4 else 0
w = W.make(name)
with er.RodBatch(w, tile_slots=tile) as b:
    b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
    b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, 1)  # one launch per step: the launches ncu captures
    b.step(spl * launches, w.dt)
    torch.cuda.synchronize()
print("ok")
