"""Raw pinned-host <-> device copy bandwidth (the PCIe ceiling of the e2e path)."""
import torch, time
n = 1 << 28  # 2 GiB of fp64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    a = time.perf_counter() - t
    t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    b = time.perf_counter() - t
    print(f"H2D {8*n/a/1e9:.1f} GB/s  D2H {8*n/b/1e9:.1f} GB/s")
