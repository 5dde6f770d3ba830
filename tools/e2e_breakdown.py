"""Where the end-to-end time goes: create (H2D + layout), steps, get_state (layout + D2H)."""
import os, sys, time, json, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2605_13766_b200 as er
w = W.make(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hp, hv, hd, ho = pin(w.positions), pin(w.velocities), pin(w.directors), pin(w.omega)
wp = dataclasses.replace(w, positions=hp.numpy(), velocities=hv.numpy(), directors=hd.numpy(), omega=ho.numpy())
outs = [torch.empty_like(x).pin_memory() for x in (hp, hv, hd, ho)]
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = er.RodBatch(wp, apply_bc_forcing=False)
    t1 = time.perf_counter()
    b.set_bc(w.clamp); b.set_forcing_from(w)
    t2 = time.perf_counter()
    b.step(100, w.dt)
    t3 = time.perf_counter()
    b.get_state_into(*[o.numpy() for o in outs])
    t4 = time.perf_counter()
    b.close()
    t5 = time.perf_counter()
    nbytes = sum(x.numel() * 8 for x in (hp, hv, hd, ho))
    print(json.dumps({"create_s": t1 - t0, "bc_forcing_s": t2 - t1, "step100_s": t3 - t2, "get_state_s": t4 - t3,
                      "destroy_s": t5 - t4, "state_GB": nbytes / 1e9}))
