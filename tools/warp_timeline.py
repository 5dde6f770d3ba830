"""Per-warp timeline of the warp-local kernel (globaltimer stamps of lane 0 for the first 64 tiles of
every warp) for one launch.  Needs a measurement build: ER_NVCC_EXTRA=-DER_TRACE=1.
Stamps: [0] before the slot wait, [1] data arrived, [2] results written to the slot, [3] after the
proxy fence + __syncwarp, [4] store issued, [5] previous store has read its slot, [6] refill issued.
Prints the mean duration of each phase and the loop period in ns."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2605_13766_b200 as er
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
spl = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = W.make(name)
with er.RodBatch(w) as b:
    b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
    b.step(3 * spl, w.dt)
    rows = 148 * 2 * 8
    tr = torch.zeros((rows, 64, 8), dtype=torch.int64, device="cuda")
    er.er_set_trace(b.handle, tr.data_ptr())
    b.step(spl, w.dt)
    er.er_set_trace(b.handle, None)
    a = tr.cpu().numpy().astype(np.uint64)
valid = a[:, :, 6] > 0
t = (a & np.uint64((1 << 48) - 1)).astype(np.int64)
t = t - t[valid][:, 0].min()
names = ["wait", "compute", "fence+syncwarp", "store issue", "wait read", "refill issue"]
per = (t[:, 1:, 0] - t[:, :-1, 0])[valid[:, 1:]]
out = {"warps": int(valid.any(1).sum()), "iters": int(valid.sum()), "period_ns": float(per.mean())}
for k, nm in enumerate(names):
    d = (t[:, :, k + 1] - t[:, :, k])[valid]
    out[nm] = {"mean": float(d.mean()), "p10": float(np.percentile(d, 10)), "p90": float(np.percentile(d, 90))}
print(json.dumps(out, indent=1))
