"""Overlap curve: ms/step of the persistent kernel vs steps per launch (memory per step 1/k)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2605_13766_b200 as er
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
tiles = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
w = W.make(name)
st = torch.cuda.Stream()
for tile in tiles:
    for spl in (1, 2, 3, 4, 8, 100):
        with er.RodBatch(w, stream=st, tile_slots=tile) as b:
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
            n = 200 if spl < 100 else 200
            b.step(spl, w.dt)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(st); b.step(n, w.dt); e1.record(st); torch.cuda.synchronize()
            print(json.dumps({"tile": tile, "spl": spl, "ms_per_step": e0.elapsed_time(e1) / n}), flush=True)
