"""Where do inter-kernel gaps come from?  cfg3: warm-up, then er_step(300) x 4 timed with events,
with and without a background nvidia-smi sampler (bench.py's ClockSampler)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W, paper_2605_13766_b200 as er
import bench
w = W.make("cfg3")
st = torch.cuda.Stream()
b = er.RodBatch(w, stream=st)
b.step(20, w.dt); torch.cuda.synchronize()
def timed(n, label):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0.record(st); b.step(n, w.dt); e1.record(st); torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / n:.4f} ms/step (host {1e3 * (time.perf_counter() - t0) / n:.4f})", flush=True)
for k in range(3):
    timed(300, f"plain #{k}")
b.set_option(er.ER_OPT_PHASE_TIMING, 1)
for k in range(2):
    timed(300, f"phase-timed #{k}")
    ph = b.phase_times(); print("   kernel ms/launch", ph.step_kernel_ms / max(ph.step_kernel_launches, 1))
with bench.ClockSampler(0) as clk:
    time.sleep(0.3)
    for k in range(3):
        timed(300, f"phase-timed + sampler #{k}")
print(clk.summary())
