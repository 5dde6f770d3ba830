"""Quick device timing of er_step on a config (development aid; bench.py is the contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2605_13766_b200 as er

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
spl = int(sys.argv[3]) if len(sys.argv) > 3 else 1
t0 = time.time(); w = W.make(name); print(f"gen {time.time()-t0:.1f}s", flush=True)
stream = torch.cuda.Stream()
b = er.RodBatch(w, stream=stream)
if spl > 1: b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
info = b.info()
print("tiles", info.n_tiles, "slots", info.tile_slots, "bytes/step", info.bytes_per_step)
b.step(5, w.dt)
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s0.record(stream); b.step(steps, w.dt); s1.record(stream); torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / steps
rate = w.n_elems_total / (ms * 1e-3)
print(f"{name}: {ms:.4f} ms/step  {rate:.4e} el-steps/s  HBM {info.bytes_per_step/(ms*1e-3)/1e9:.1f} GB/s (B_min)")
if getattr(w, "contact", None) is not None:
    st = b.contact_stats()
    print({k: getattr(st, k) for k, _ in st._fields_})
