"""Benchmark: rod element-updates/s (fp64) of the batched Cosserat rod step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3] [--steps-per-launch S] [--scaling strong|weak]

One bench "step" = one position-Verlet time step (all SURVEY §8(a) rows A1-A10) over the
whole batch.  Default workload: BASELINE.json configs[2] ("cfg3": 1,048,576 rods x 16
elements, the paper's 1024^2-filament size), synthetic and seeded (workloads/).
Multi-GPU: one process per GPU, launched by torchrun or, when `--gpus N` is given without a
torchrun environment (no WORLD_SIZE), spawned by bench.py itself (N ranks, NCCL, rendezvous on
127.0.0.1).  The default is strong scaling -- the one cfg3 batch of 1,048,576 rods sharded into
slot-balanced contiguous rod ranges (BASELINE configs[2] "sharded over 1/2/4/8 GPUs", the paper's
strong-scaling experiment); `--scaling weak` gives every rank its own full batch.
Rods are independent, so there is no data-path collective: NCCL all-reduces only the scalar
diagnostics, once, after the timed region.  Rank 0 prints one JSON line with the per-rank times
and shard sizes.

`--impl reference`: there is no reference implementation to install (the paper ships no
code); the reference arm is the CPU oracle (oracle/, plain C fp64), timed on
the host on a bounded rod sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=list(W.CONFIG_NAMES) + list(W.EXTRA_CONFIGS))
    ap.add_argument("--sweeps", type=int, default=0,
                    help="ER_OPT_SWEEPS_PER_LAUNCH (0 = the library default)")
    ap.add_argument("--steps-per-launch", type=int, default=1,
                    help="1 = every step streams the state through HBM (the B_min design); "
                         ">1 = temporal blocking (SURVEY NEXT-1)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-fanout", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-temporal", action="store_true")
    ap.add_argument("--no-contact", action="store_true")
    ap.add_argument("--cpu-sample-rods", type=int, default=8192)
    ap.add_argument("--cpu-sample-steps", type=int, default=400)
    return ap.parse_args()


def peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def b_min_per_el_step(w, q_planes: float = 9.0, rec_bytes: float = 128.0) -> float:
    """SURVEY §8 D.3 with the stored director form (DESIGN §4 "Director storage"): the state is
    r, v per node and d1, d2, w per element (d3 = d1 x d2 is rebuilt on chip), so
    16 [6(N+1) + 9 N] + P + 24 (N-1) chi_kappa0 bytes per rod-step, / N (SURVEY's 12 N counts
    the full 3x3 Q; `b_min_survey_3x3` below keeps that figure for reference).
    Contact mode (NEXT-4) adds, for the step kernel: the contact force on each element's
    two nodes read (48 B per element), the node records for the next contact evaluation written
    (48 B per node) and the build positions read for the Verlet check (24 B per node).
    `rec_bytes` is SURVEY's P, the per-rod record (128 B); a shared-material batch (every rod has
    the same material constants; er_info.shared_material) needs only its 48-byte rod
    record (tip force, actuation, flags) per rod-step."""
    N = w.n_elems.astype(np.float64)
    per_rod = 16.0 * (6.0 * (N + 1) + q_planes * N) + rec_bytes + (24.0 * (N - 1) if w.rest_kappa is not None else 0.0)
    if getattr(w, "contact", None) is not None:
        per_rod = per_rod + 48.0 * N + 72.0 * (N + 1)
    return float(per_rod.sum() / N.sum())


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def _nvml_loop(self, period):
        import pynvml as N
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
        while not self.stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            ev = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append([str(self.index), str(sm), str(mx), "", hex(ev)]
                             + ["Active" if ev & b else "Not Active" for b in bits])
            self.stop.wait(period)

    def __enter__(self):
        try:
            if os.environ.get("ER_BENCH_NO_CLOCKS"):  # measurement of the sampler's own effect
                raise RuntimeError("clock sampling disabled")
            if os.environ.get("ER_BENCH_CLOCKS", "smi") == "nvml":
                # ER_BENCH_CLOCKS=nvml: in-process NVML (clock + event-reason queries only) instead of
                # the recipe's nvidia-smi loop; both stall the GPU's kernel launches now and then
                # (DESIGN §4 "Monitoring stalls")
                import pynvml as N
                N.nvmlInit()
                self.stop = threading.Event()
                self.th = threading.Thread(target=self._nvml_loop,
                                           args=(float(os.environ.get("ER_BENCH_CLOCK_MS", "200")) / 1e3,), daemon=True)
                self.th.start()
                self.nvml = True
                return self
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("ER_BENCH_CLOCK_MS", "200")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if getattr(self, "nvml", False):
            self.stop.set()
            self.th.join(timeout=5)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def shard(w, rank, world, scaling):
    """Strong: contiguous rod ranges balanced by slot count (N_r + 1).  Weak: every rank a full
    copy-size batch (rank-seeded sample order is irrelevant: rods are independent)."""
    if world == 1 or scaling == "weak":
        return w
    slots = np.cumsum(w.n_elems.astype(np.int64) + 1)
    total = slots[-1]
    cuts = [0] + [int(np.searchsorted(slots, total * k / world, side="left")) + 1 for k in range(1, world)] + [w.n_rods]
    if getattr(w, "contact", None) is not None:
        # rods that touch must stay on one GPU: cut only between the fibres stacks, which never
        # touch (0.2 L apart), so the shards need no halo exchange
        per = W.FIBRES["layers"] * W.FIBRES["per_layer"]
        cuts = [int(round(c / per)) * per for c in cuts]
    cuts = np.clip(cuts, 0, w.n_rods)
    return w.subset(np.arange(cuts[rank], cuts[rank + 1]))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(w, n_rods, n_steps, seed=3):
    """The oracle as it stands (single-threaded C), on a seeded rod sample (for contact workloads:
    the first whole stack, an independent sub-problem), pinned to one host core while it runs
    (taskset)."""
    import oracle
    if getattr(w, "contact", None) is not None:
        rods = np.arange(min(w.n_rods, W.FIBRES["layers"] * W.FIBRES["per_layer"]))
    else:
        rods = W.sample_rods(w, n_rods, seed=seed)
    ws = w.subset(rods)
    aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    if aff:
        os.sched_setaffinity(0, {min(aff)})
    try:
        t0 = time.perf_counter()
        st, s, _, _ = oracle.step(ws, n_steps=n_steps)
        dt = time.perf_counter() - t0
    finally:
        if aff:
            os.sched_setaffinity(0, aff)
    return ws.n_elems_total * n_steps / dt, dt, ws


def _fanout_worker(args):
    ws, n_steps = args
    import oracle
    t0 = time.perf_counter()
    oracle.step(ws, n_steps=n_steps)
    return ws.n_elems_total * n_steps, time.perf_counter() - t0


def oracle_fanout_rate(w, rods_per_proc, n_steps, seed=5):
    """SURVEY §8(d) whole-host fan-out: the oracle as it stands in one process per host core,
    each on its own seeded rod shard (rods are independent).  Rate = all element-steps / the
    slowest process's time."""
    import multiprocessing as mp
    import oracle
    oracle.build()            # once, in the parent: the spawned workers only dlopen it
    n_proc = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    rods = W.sample_rods(w, min(w.n_rods, rods_per_proc * n_proc), seed=seed)
    shards = [w.subset(np.sort(part)) for part in np.array_split(rods, n_proc) if len(part)]
    with mp.get_context("spawn").Pool(len(shards)) as pool:
        res = pool.map(_fanout_worker, [(x, n_steps) for x in shards])
    work = sum(r[0] for r in res)
    slow = max(r[1] for r in res)
    return {"value": work / slow, "unit": "element-steps/s", "cores": len(shards), "kind": "oracle, one process per core",
            "sample": f"{len(rods)} seeded rods of the workload in {len(shards)} shards x {n_steps} steps "
                      f"({work:.3g} element-steps, slowest process {slow:.1f} s)"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = W.make(a.config)
    import oracle
    if getattr(w, "contact", None) is not None:   # a whole stack: an independent contact sub-problem
        rods = np.arange(min(w.n_rods, W.FIBRES["layers"] * W.FIBRES["per_layer"]))
    else:
        rods = W.sample_rods(w, min(4096, w.n_rods), seed=4)
    ws = w.subset(rods)
    st = oracle.State.of(ws)
    for _ in range(max(a.warmup, 0)):
        oracle.step(ws, st, n_steps=1)
    steps = max(1, min(a.steps, 20))
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.step(ws, st, n_steps=1)
    dt = time.perf_counter() - t0
    value = ws.n_elems_total * steps / dt
    sample = f"{len(rods)} seeded rods of {a.config} ({ws.n_elems_total} elements) x {steps} steps per run"
    print(json.dumps({
        "impl": "reference", "metric": "rod element-updates/sec (fp64)", "value": value,
        "unit": "element-steps/s", "n_gpus": a.gpus, "steps": steps, "warmup": a.warmup,
        "ms_per_step": dt / steps * 1e3, "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, workloads/)",
        "config": {"workload": f"{a.config}: {w.n_rods} rods (sample of {len(rods)})", "sample_rods": len(rods)},
        "cpu_baseline": {"value": value, "unit": "element-steps/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "element-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "no reference code exists (SURVEY §0); the reference arm is the CPU oracle on the host",
    }), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _spawned_rank(rank, world, port, argv):
    """Child process of `bench.py --gpus N` run without torchrun: the torchrun environment, then
    the ordinary per-rank path."""
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.argv = argv
    main()


def spawn_ranks(a):
    """`--gpus N` without a torchrun environment: start N ranks here (one process per GPU)."""
    import torch.multiprocessing as mp
    os.environ.setdefault("NCCL_DEBUG", "INFO")             # communicator init (nranks) in the log
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    mp.start_processes(_spawned_rank, args=(a.gpus, _free_port(), list(sys.argv)), nprocs=a.gpus,
                       join=True, start_method="spawn")


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(a)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and rank == 0:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
    # ER_BENCH_SHARE_GPU=1: functional test of the multi-rank path on a one-GPU box (ranks share
    # GPU 0 and reduce over gloo) -- never a measurement
    share = os.environ.get("ER_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2605_13766_b200 as er

    wfull = W.make(a.config)
    w = shard(wfull, rank, world, a.scaling)
    stream = torch.cuda.Stream(device=local)
    b = er.RodBatch(w, device=local, stream=stream)
    if a.steps_per_launch > 1:
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, a.steps_per_launch)
    if a.sweeps > 0:
        b.set_option(er.ER_OPT_SWEEPS_PER_LAUNCH, a.sweeps)
    dt = w.dt

    # warm-up (untimed)
    b.step(a.warmup, dt)
    torch.cuda.synchronize()
    launches0 = b.info().launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b.set_option(er.ER_OPT_PHASE_TIMING, 1)  # CUDA events around every step-kernel launch (own stream)
    with ClockSampler(local) as clk:
        time.sleep(0.3)                     # let the sampler start
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        b.step(a.steps, dt)                 # K launches of the fused step on `stream`
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = b.info().launches - launches0
    ph = b.phase_times()
    b.set_option(er.ER_OPT_PHASE_TIMING, 0)
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    per_rank = [{"rank": rank, "ms_per_step": ms / a.steps, "rods": w.n_rods, "elements": w.n_elems_total,
                 "device": local}]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank[0])
        per_rank = gathered
    el_local = w.n_elems_total
    el_total = torch.tensor([float(el_local)], dtype=torch.float64, device=f"cuda:{local}")
    # scalar diagnostics: the only cross-GPU exchange (NCCL all-reduce of ~12 fp64)
    diag = torch.tensor(b.diagnostics(), dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        vmax = diag[9].clone()
        dist.all_reduce(el_total)
        dist.all_reduce(diag)
        dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
        diag[9] = vmax
    value = float(el_total.item()) * a.steps / (ms_max * 1e-3)

    # roofline of the dominant kernel (the rod step kernel; in contact mode the step kernel beside
    # the contact graph): algorithmic bytes per launch / its mean launch duration from the CUDA
    # events er_step records around each launch on its stream (ER_OPT_PHASE_TIMING)
    shared = bool(b.info().shared_material)
    bmin = b_min_per_el_step(w, rec_bytes=48.0 if shared else 128.0)
    per_launch_bytes = bmin * el_local * max(1, a.steps_per_launch)
    n_kl = max(int(ph.step_kernel_launches), 1)
    launch_ms = ph.step_kernel_ms / n_kl if ph.step_kernel_launches else ms / max(launches, 1)
    achieved = per_launch_bytes / (launch_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            key = f"{a.config}_spl{a.steps_per_launch}"
            if key in tj:
                traffic = tj[key]["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": peak_src, "bytes_per_el_step": bmin,
            "b_min_survey_3x3": b_min_per_el_step(w, 12.0), "b_min_survey_P128": b_min_per_el_step(w),
            "shared_material": shared,
            "kernel": (f"er::pair_bulk<FEAT,{b.info().warp_buffers}> (warp-pair step: lane = element, a rod on "
                       "the 64 lanes of two warps, per-pair TMA bulk load/store ring)" if b.info().warp_rod_elems > 32
                       else f"er::warp_bulk<FEAT,{b.info().warp_buffers},{b.info().warp_rod_elems}> (warp-local step: "
                       "lane = element, shuffle exchanges, per-warp TMA bulk load/store ring)" if b.info().warp_rod_elems
                       else f"er::fused_persistent<{b.info().tile_slots},MINB,FEAT> (tile step, CTA-level TMA bulk "
                            "load/store pipeline)"),
            "kernel_ms_per_launch": launch_ms, "kernel_share_of_step": ph.step_kernel_ms / ms if ms > 0 else None}
    if ph.contact_evals:
        roof["contact_ms_per_step"] = ph.contact_ms / ph.contact_evals
    if a.steps_per_launch > 1:
        roof["note"] = ("temporal blocking: the state crosses HBM once per launch of "
                        f"{a.steps_per_launch} steps, so 'achieved' counts B_min per step and can exceed the "
                        "HBM peak; the binding resource is the FP64 pipe")

    # NEXT-1 context: the same job with the rod tile kept on chip for several steps per launch
    # (temporal blocking; bitwise-identical results), timed the same way on the same batch
    temporal = None
    if a.steps_per_launch == 1 and not a.no_temporal and getattr(w, "contact", None) is None:
        spl = 100
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, spl)
        b.step(spl, dt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b.step(a.steps, dt)
        e1.record(stream)
        torch.cuda.synchronize()
        tms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        b.set_option(er.ER_OPT_STEPS_PER_LAUNCH, 1)
        temporal = {"steps_per_launch": spl, "ms_per_step": float(tms.item()) / a.steps,
                    "value": float(el_total.item()) * a.steps / (float(tms.item()) * 1e-3),
                    "note": "SURVEY NEXT-1: state crosses HBM once per launch; FP64/issue-bound"}
        tpath = os.path.join(ROOT, "profiles", "temporal.json")
        try:  # the FP64-pipe share SURVEY NEXT-1 asks for, from the committed ncu capture
            tj = json.load(open(tpath)).get(f"{a.config}_spl{spl}")
            if tj:
                temporal["fp64_pipe_pct_of_peak"] = tj["fp64_pipe_pct_of_peak"]
                temporal["issue_active_pct"] = tj["issue_active_pct"]
                temporal["fp64_source"] = tj["source"]
        except Exception:
            pass

    # NEXT-4 context: the contact workload (fibres: 65,536 rods x 16 elements in crossed layers,
    # HHG broad phase + Verlet lists + narrow phase every step), same timing protocol
    contact = None
    if world == 1 and not a.no_contact and a.config != "fibres":
        contact = contact_run(er, a.steps, local, stream)

    # end-to-end through the public API with HOST buffers (pinned): create from host, K steps,
    # state back to host; the H2D/D2H bytes are amortised over the K steps of the job
    e2e = None
    if not a.no_e2e:
        e2e = e2e_run(er, w, a.steps, dt, local, world)

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu_baseline:
            cs = a.cpu_sample_steps if getattr(wfull, "contact", None) is None else max(5, a.cpu_sample_steps // 6)
            rate, secs, ws = oracle_rate(wfull, a.cpu_sample_rods, cs)
            what = "seeded rods" if getattr(wfull, "contact", None) is None else "rods (one whole stack, exhaustive contact search)"
            cpu = {"value": rate, "unit": "element-steps/s", "cores": 1, "kind": "oracle", "cpu": cpu_model(),
                   "sample": f"{ws.n_rods} {what} of {a.config} x {cs} steps "
                             f"({ws.n_elems_total * cs:.3g} element-steps, {secs:.1f} s, 1 thread pinned to one core)"}
            if not a.no_cpu_fanout and getattr(wfull, "contact", None) is None:
                try:
                    cpu["fanout"] = oracle_fanout_rate(wfull, 512, a.cpu_sample_steps)
                except Exception as ex:  # the single-thread figure stands on its own
                    cpu["fanout"] = {"unavailable": str(ex)[:200]}
        out = {
            "metric": "rod element-updates/sec (fp64)", "value": value, "unit": "element-steps/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max / a.steps,
            "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, workloads/)",
            "config": {"workload": f"{a.config}: {wfull.n_rods} rods x "
                                   f"{int(wfull.n_elems.min())}-{int(wfull.n_elems.max())} elements "
                                   f"({wfull.n_elems_total} elements), dt={wfull.dt}",
                       "rods_per_gpu": w.n_rods, "elements_per_gpu": w.n_elems_total,
                       "steps_per_launch": a.steps_per_launch,
                       "sweeps_per_launch": a.sweeps or er.ER_DEFAULT_SWEEPS,
                       "l2": "inputs larger than L2 (state %.2f GB per GPU vs 126 MB L2)" % (
                           b.info().device_bytes / 1e9),
                       "parallelism": (f"weak: each of {world} GPU(s) advances its own {a.config} batch"
                                       if a.scaling == "weak" else f"strong: one {a.config} batch in rod shards over "
                                       f"{world} GPU(s)") + "; NCCL for scalar diagnostics only"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "per_rank": per_rank,
            "temporal_blocking": temporal,
            "contact": contact,
            "clocks": clk.summary(),
            "paper_context": PAPER_CONTEXT,
            "diagnostics": {k: float(v) for k, v in zip(er.DIAG_NAMES, diag.cpu().numpy())},
        }
        print(json.dumps(out), flush=True)
    b.close()
    if world > 1:
        dist.destroy_process_group()


def contact_run(er, steps, local, stream):
    import torch
    wc = W.make("fibres")
    bc = er.RodBatch(wc, device=local, stream=stream)
    bc.step(20, wc.dt)
    torch.cuda.synchronize()
    l0 = bc.info().launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    bc.step(steps, wc.dt)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = bc.contact_stats()
    launches = bc.info().launches - l0
    bc.close()
    return {"workload": f"fibres: {wc.n_rods} rods x 16 elements ({wc.n_elems_total} elements) in crossed layers "
                        "on a floor, contact + friction every step, dt=1e-6",
            "ms_per_step": ms / steps, "value": wc.n_elems_total * steps / (ms * 1e-3), "unit": "element-steps/s",
            "contacts": st.contacts, "plane_contacts": st.plane_contacts, "candidates": st.candidates,
            "list_builds": st.builds, "gpu_launches": launches,
            "note": "SURVEY NEXT-4: HHG broad phase with Verlet lists (device-side rebuild), exact "
                    "segment-segment narrow phase; one CUDA graph + one persistent step kernel per step"}


# The paper's own performance figures (CPU only; no absolute throughput is printed), quoted with their
# hardware as context beside this run (north_star) -- not targets, not ratios.
PAPER_CONTEXT = {
    "so3_rotation_kernel": "~0.7 -> ~20 GFLOP/s fp64 after SoA2AoS + SIMD + blocking, 95% of single-core peak, "
                           "Intel Core i9-11900K, one core (PAPER.md:30-32, :44-45)",
    "strong_scaling": "'near-optimal' with the asynchronous protocol for 1024^2 filaments, up to 64 AMD EPYC 7742 "
                      "on SDSC Expanse; no absolute step times printed (PAPER.md:33-34, :46-49)",
}


def e2e_run(er, w, steps, dt, local, world):
    import torch
    import dataclasses
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hp, hv, hd, ho = pin(w.positions), pin(w.velocities), pin(w.directors), pin(w.omega)
    wp = dataclasses.replace(w, positions=hp.numpy(), velocities=hv.numpy(), directors=hd.numpy(), omega=ho.numpy())
    outp, outv = torch.empty_like(hp).pin_memory(), torch.empty_like(hv).pin_memory()
    outd, outo = torch.empty_like(hd).pin_memory(), torch.empty_like(ho).pin_memory()
    # one untimed warm-up job on the same pinned buffers (3 steps): the first job of a process pays
    # one-time costs (first DMA from freshly pinned pages, first allocations and module loads:
    # create 0.68 s vs 0.15 s, profiles/r02/e2e_phases_r02d.log), like the warm-up steps of `value`
    bw = er.RodBatch(wp, device=local)
    bw.step(3, dt)
    bw.get_state_into(outp.numpy(), outv.numpy(), outd.numpy(), outo.numpy())
    bw.close()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    b = er.RodBatch(wp, device=local)                  # H2D of the inputs (pinned host)
    t1 = time.perf_counter()
    b.step(steps, dt)
    t2 = time.perf_counter()
    b.get_state_into(outp.numpy(), outv.numpy(), outd.numpy(), outo.numpy())  # D2H of the result
    t3 = time.perf_counter()
    secs = t3 - t0
    b.close()
    tt = torch.tensor([secs], dtype=torch.float64, device=f"cuda:{local}")
    el = torch.tensor([float(w.n_elems_total)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(el)
    state_bytes = 8 * (w.positions.size + w.velocities.size + w.directors.size + w.omega.size)
    param_bytes = 8 * (w.rest_lengths.size + 7 * w.n_rods) + 4 * w.n_rods
    return {"value": float(el.item()) * steps / float(tt.item()), "unit": "element-steps/s",
            "h2d_bytes_per_step": (state_bytes + param_bytes) / steps, "d2h_bytes_per_step": state_bytes / steps,
            "seconds": float(tt.item()),
            "phases_s": {"create": t1 - t0, "step": t2 - t1, "get_state": t3 - t2},
            "what": f"er_create_batch from pinned host arrays + er_step({steps}) + er_get_state to pinned host, "
                    "wall clock (max over ranks), after one untimed 3-step warm-up job on the same pinned buffers; "
                    "transfer bytes are per job / steps"}


if __name__ == "__main__":
    main()
