"""Kernel ablation on one config: persistent fused (kind 0), one-tile-per-CTA fused (2),
staged three launches (1), and temporal blocking.  Device time with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, torch
import workloads as W
import paper_2605_13766_b200 as er

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
tiles = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else None
w = W.make(name)
stream = torch.cuda.Stream()
res = {}
for tile in tiles:
  for label, kernel, spl in (("persistent", 0, 1), ("one_tile_per_cta", 2, 1), ("staged_3_launch", 1, 1),
                             ("persistent_spl10", 0, 10), ("persistent_spl100", 0, 100), ("memory_probe", 3, 1)):
    if kinds and label not in kinds:
        continue
    label = f"{label}[tile={tile}]"
    with er.RodBatch(w, stream=stream, tile_slots=tile) as b:
        b.set_option(er.ER_OPT_KERNEL, kernel)
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
        b.step(spl if spl > 1 else 5, w.dt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream); b.step(steps, w.dt); e1.record(stream); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        info = b.info()
        res[label] = {"ms_per_step": ms, "el_steps_per_s": w.n_elems_total / (ms * 1e-3),
                      "bmin_GBps": info.bytes_per_step / (ms * 1e-3) / 1e9}
        print(label, json.dumps(res[label]), flush=True)
