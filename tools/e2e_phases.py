"""Time the phases of one end-to-end cfg3 job (create from pinned host arrays, 1000 steps, state back to pinned host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, dataclasses
import workloads as W, paper_2605_13766_b200 as er
w = W.make("cfg3")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hp, hv, hd, ho = pin(w.positions), pin(w.velocities), pin(w.directors), pin(w.omega)
wp = dataclasses.replace(w, positions=hp.numpy(), velocities=hv.numpy(), directors=hd.numpy(), omega=ho.numpy())
outs = [torch.empty_like(x).pin_memory() for x in (hp, hv, hd, ho)]
for rep in range(int(os.environ.get("REPS", "2"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = er.RodBatch(wp)
    t1 = time.perf_counter()
    b.step(1000, w.dt)
    t2 = time.perf_counter()
    b.get_state_into(*[o.numpy() for o in outs])
    t3 = time.perf_counter()
    b.close()
    print(f"create {t1-t0:.3f} s  step {t2-t1:.3f} s  get_state {t3-t2:.3f} s", flush=True)
