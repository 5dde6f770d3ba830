"""Device time of the non-step API calls on a BASELINE config (development aid): create (from device
arrays), get_state into device arrays, diagnostics -- CUDA events on the batch stream.
    python tools/api_phases.py cfg3"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses
import torch
import workloads as W
import paper_2605_13766_b200 as er
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = W.make(name)
wd = dataclasses.replace(w, **{k: torch.tensor(getattr(w, k), device="cuda") for k in ("positions", "velocities", "directors", "omega")})
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b = er.RodBatch(wd)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    outs = [torch.empty_like(getattr(wd, k)) for k in ("positions", "velocities", "directors", "omega")]
    b.step(2, w.dt)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    b.get_state_into(*outs)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    d = b.diagnostics()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"{name} rep {rep}: create {1e3*(t1-t0):.1f} ms, get_state {1e3*(t3-t2):.2f} ms, diagnostics {1e3*(t4-t3):.2f} ms "
          f"(warp N={b.info().warp_rod_elems}, tiles {b.info().n_tiles})", flush=True)
    b.close()
