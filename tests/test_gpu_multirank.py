"""Multi-rank product path on the GPU: rods sharded over ranks, one process per rank.

The round's GPU boxes have one B200, so the ranks share GPU 0 and reduce over gloo; that checks the
sharding, the per-rank batches and bench.py's multi-rank harness through the product path (the C-ABI
library in every rank), not NCCL performance.  Rods are independent, so each shard's trajectory must
equal, bitwise, the same rods of the single-rank run.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import bench
import workloads as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def er():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_13766_b200 as er
    return er


def _rank(rank, world, port, name, n_rods, n_steps, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2605_13766_b200 as er
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = W.make(name, n_rods=n_rods)
    ws = bench.shard(w, rank, world, "strong")
    with er.RodBatch(ws, device=0) as b:
        b.step(n_steps, ws.dt)
        pos, vel, dirs, om, t = b.get_state()
        d = torch.tensor(b.diagnostics(), dtype=torch.float64)
    e = d[:9].clone()
    dist.all_reduce(e)                                        # the scalar diagnostics exchange
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pos=pos, vel=vel, dirs=dirs, om=om, t=t,
             n_rods=ws.n_rods, diag_sum=e.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n_rods,world", [("cfg5", 3000, 2), ("cfg3", 20000, 3)])
def test_shards_equal_single_rank_bitwise(er, tmp_path, name, n_rods, world):
    import torch.multiprocessing as mp
    n_steps = 40
    port = bench._free_port()
    mp.start_processes(_rank, args=(world, port, name, n_rods, n_steps, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    w = W.make(name, n_rods=n_rods)
    with er.RodBatch(w) as b:
        b.step(n_steps, w.dt)
        full = b.get_state()
        dfull = b.diagnostics()
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    assert sum(int(p["n_rods"]) for p in parts) == w.n_rods
    assert all(int(p["n_rods"]) > 0 for p in parts)
    for k, key in enumerate(("pos", "vel", "dirs", "om")):
        assert np.array_equal(np.concatenate([p[key] for p in parts]), full[k]), key
    assert all(float(p["t"]) == full[4] for p in parts)
    # all-reduced energies/momentum equal the single-rank sums up to summation order
    ds = parts[0]["diag_sum"]
    assert np.allclose(ds[:6], dfull[:6], rtol=1e-12, atol=0)


def test_bench_spawns_ranks_strong_scaling():
    """`bench.py --gpus 2` without torchrun starts two ranks itself; the default is strong scaling
    of cfg3: the shards' rods add up to the 1,048,576 rods of BASELINE configs[2]."""
    env = dict(os.environ, ER_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "5",
                        "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-temporal", "--no-contact"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    assert len(out["per_rank"]) == 2
    assert sum(r["rods"] for r in out["per_rank"]) == 1024 * 1024
    assert sum(r["elements"] for r in out["per_rank"]) == 16 * 1024 * 1024
    assert out["value"] > 0
