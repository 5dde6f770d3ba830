"""Strong-scaling proxy on one GPU: per-step time of the cfg3 shard one rank owns at N = 1, 2, 4, 8
(1,048,576 / N rods), run alone.  rate_N / (N rate_1) is the best 8-GPU efficiency the kernel
allows (no communication is on the step path).   python tools/shard_eff.py [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2605_13766_b200 as er
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
wfull = W.make("cfg3")
stream = torch.cuda.Stream()
res = {}
for rep in range(2):
    for n in (1, 2, 4, 8):
        w = bench.shard(wfull, 0, n, "strong")
        b = er.RodBatch(w, stream=stream)
        b.step(20, w.dt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream); b.step(steps, w.dt); e1.record(stream); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rate = w.n_elems_total / (ms * 1e-3)
        res[n] = rate
        inf = b.info()
        print(f"N={n} rods {w.n_rods}: {ms*1e3:.1f} us/step, {rate:.3g} el-steps/s per GPU, "
              f"eff {rate / res[1]:.3f} (warp N={inf.warp_rod_elems}, tiles {inf.n_tiles})", flush=True)
        b.close()
