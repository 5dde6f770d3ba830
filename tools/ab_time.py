"""A/B device timing of er_step variants on one config (development aid):
    python tools/ab_time.py cfg3 300 0 4   # ER_OPT_KERNEL values to compare
    ER_TILE=128 python tools/ab_time.py cfg3 300 0"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2605_13766_b200 as er

name, steps = sys.argv[1], int(sys.argv[2])
kernels = [int(k) for k in sys.argv[3:]] or [0]
w = W.make(name)
stream = torch.cuda.Stream()
b = er.RodBatch(w, stream=stream, tile_slots=int(os.environ.get("ER_TILE", "0")))
if os.environ.get("ER_SWEEPS"):
    b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, int(os.environ["ER_SWEEPS"]))
for rep in range(3):
    for k in kernels:
        b.set_option(er.ER_OPT_KERNEL, k)
        b.step(10, w.dt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream); b.step(steps, w.dt); e1.record(stream); torch.cuda.synchronize()
        print(f"{name} kernel={k} rep={rep}: {e0.elapsed_time(e1) / steps:.4f} ms/step", flush=True)
