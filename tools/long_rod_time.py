"""Device timing of long rods (16,384 rods x 1000 elements: thread-block clusters), 1 and 10 steps per launch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_2605_13766_b200 as er
# cfg3-like rods but N = 1000 (L = 6.25 m? keep lhat = 0.00625, r = 1e-3), 16384 rods = 16.4 M elements
R, N = 16384, 1000
n = np.full(R, N, np.int32); lh = np.full(R, 0.00625)
mat = W._rod_material(R, 1e-3, 1e6)
rng = np.random.default_rng(0)
Q0 = W.uniform_so3(rng, R)
pos = W.straight_rods(n, lh, np.zeros((R, 3)), Q0[:, 2, :])
w = W.Workload("long", n, W._expand(lh, n), **mat, positions=pos, velocities=np.zeros_like(pos),
               directors=W._expand(Q0, n), omega=np.zeros((R * N, 3)), clamp=np.zeros(R, np.int8),
               gravity=np.zeros(3), damping=np.full(R, 0.1), tip_force=rng.normal(0, 1e-6, (R, 3)), dt=1e-6)
st = torch.cuda.Stream()
b = er.RodBatch(w, stream=st)
print("tiles", b.info().n_tiles)
for spl in (1, 10):
    b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
    b.step(20, w.dt); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); b.step(200, w.dt); e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    el = R * N
    bmin = (16 * (6 * (N + 1) + 9 * N) + 128) / N  # stored state: r, v, d1, d2, w
    print(f"spl={spl}: {ms:.4f} ms/step  {el / (ms * 1e-3):.3e} el-steps/s  {bmin * el / (ms * 1e-3) / 1e9:.0f} GB/s (B_min)")
