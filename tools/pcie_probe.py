"""PCIe probe: pinned H2D bandwidth of a dataset-sized buffer, alone and
concurrent with a compute stream; D2H of a hot-table-sized result."""
import time
import torch
dev = torch.device("cuda", 0)
n = 4_812_807_872 // 4
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device=dev)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D pinned {h.numel()*4/1e9:.2f} GB in {dt*1e3:.1f} ms = {h.numel()*4/dt/1e9:.1f} GB/s")
w = torch.empty(2_075_123 * 16, device=dev)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    o = w.cpu(); dt = time.perf_counter() - t
    print(f"D2H .cpu() {w.numel()*4/1e6:.0f} MB in {dt*1e3:.1f} ms = {w.numel()*4/dt/1e9:.1f} GB/s")
ph = torch.empty(w.numel()).pin_memory()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    ph.copy_(w, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"D2H pinned {w.numel()*4/1e6:.0f} MB in {dt*1e3:.1f} ms = {w.numel()*4/dt/1e9:.1f} GB/s")
