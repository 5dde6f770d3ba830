import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_2605_13766_b200 as er
w = W.make("cfg5")
ws = w.subset(np.nonzero(w.n_elems <= 255)[0])
print("rods", w.n_rods, "->", ws.n_rods)
for tile in (512, 256, 512, 256):
    st = torch.cuda.Stream()
    with er.RodBatch(ws, stream=st, tile_slots=tile) as b:
        b.step(10, ws.dt); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); b.step(100, ws.dt); e1.record(st); torch.cuda.synchronize()
        print(tile, b.info().n_tiles, f"{e0.elapsed_time(e1)/100:.4f} ms/step", flush=True)
