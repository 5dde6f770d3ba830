"""Interleaved device timing of the warp-local kernel against the tile kernel (development aid).
    python tools/warp_ab.py cfg3 300 "" "ER_NO_WARP=1" "ER_WARP_TILE_RODS=15" "ER_WARP_BUFFERS=2"
Each argument after the step count is a space-separated set of environment settings applied while
the batch is created (they select the layout / kernel); "" = the defaults.  SPL=k in a setting runs
k steps per launch (temporal blocking)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2605_13766_b200 as er

name, steps = sys.argv[1], int(sys.argv[2])
variants = sys.argv[3:] or [""]
w = W.make(name)
stream = torch.cuda.Stream()
for rep in range(3):
    for v in variants:
        env = dict(kv.split("=", 1) for kv in v.split())
        spl = int(env.pop("SPL", "1"))
        sweeps = int(env.pop("SWEEPS", "0"))  # ER_OPT_SWEEPS_PER_LAUNCH (0 = the library's default)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        b = er.RodBatch(w, stream=stream)
        for k, x in old.items():
            if x is None:
                os.environ.pop(k)
            else:
                os.environ[k] = x
        if spl > 1:
            b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
        if sweeps:
            b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, sweeps)
        def stepq(n):  # ER_AB_IGNORE_FAULTS=1: timing experiments whose physics is knowingly wrong
            try:
                b.step(n, w.dt)
            except er.ErError:
                if not os.environ.get("ER_AB_IGNORE_FAULTS"):
                    raise
        stepq(max(10, spl))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream); stepq(steps); e1.record(stream); torch.cuda.synchronize()
        inf = b.info()
        print(f"{name} [{v or 'default'}] rep={rep}: {e0.elapsed_time(e1) / steps:.4f} ms/step "
              f"(warp N={inf.warp_rod_elems}, buffers {inf.warp_buffers}, tiles {inf.n_tiles}, block {inf.tile_slots})",
              flush=True)
        b.close()
        del b
        torch.cuda.synchronize()
