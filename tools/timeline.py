"""Per-CTA timeline of the persistent kernel (globaltimer stamps) for one launch.  Needs a
measurement build: ER_NVCC_EXTRA=-DER_TRACE=1 python paper_2605_13766_b200/build.py (the
production kernel has no timeline code; er_set_trace returns ER_EINVAL there)."""
import os, sys, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_2605_13766_b200 as er
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = W.make(name)
with er.RodBatch(w, tile_slots=tile) as b:
    b.step(3, w.dt)
    grid = 148 * 8
    tr = torch.zeros((grid, 64, 4), dtype=torch.int64, device="cuda")
    er.er_set_trace(b.handle, tr.data_ptr())
    b.step(1, w.dt)
    er.er_set_trace(b.handle, None)
    a = tr.cpu().numpy().astype(np.uint64)
valid = a[:, :, 3] > 0
sm = (a[:, :, 0] >> np.uint64(56)).astype(np.int64)
t = a & np.uint64((1 << 48) - 1)
t = t.astype(np.int64)
t0 = t[valid][:, 0].min()
t = t - t0
wait = (t[:, :, 1] - t[:, :, 0])[valid]; comp = (t[:, :, 2] - t[:, :, 1])[valid]; store = (t[:, :, 3] - t[:, :, 2])[valid]
per = (t[:, 1:, 0] - t[:, :-1, 0])[valid[:, 1:]]
print(json.dumps({"tile": tile, "ctas": int(valid.any(1).sum()), "iters": int(valid.sum()),
                  "period_ns": float(per.mean()), "wait_ns": float(wait.mean()), "compute_ns": float(comp.mean()),
                  "store_ns": float(store.mean())}))
bysm = collections.defaultdict(list)
for c in range(a.shape[0]):
    if valid[c].any(): bysm[int(sm[c, 0])].append(c)
print("ctas per sm:", collections.Counter(len(v) for v in bysm.values()))
for s_id in sorted(bysm)[:2]:
    for c in bysm[s_id]:
        row = [(int(t[c, k, 0]) // 100, int(t[c, k, 1]) // 100, int(t[c, k, 2]) // 100) for k in range(10) if valid[c, k]]
        print("sm", s_id, "cta", c, "(wait start, data, compute end) x100ns:", row)
