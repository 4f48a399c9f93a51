"""PCIe full-duplex probe: 74 MB H2D and 21 MB D2H from pinned memory, alone, one after the other, concurrently."""
import time, torch
n_h2d, n_d2h = 74147840 // 8, 20971520 // 8
hx = torch.empty(n_h2d, dtype=torch.float64, pin_memory=True); dx = torch.empty(n_h2d, dtype=torch.float64, device="cuda")
dy = torch.rand(n_d2h, dtype=torch.float64, device="cuda"); hy = torch.empty(n_d2h, dtype=torch.float64, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def seq():
    dx.copy_(hx, non_blocking=True); hy.copy_(dy, non_blocking=True)
def par():
    with torch.cuda.stream(s1): dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2): hy.copy_(dy, non_blocking=True)
for name, f in (("h2d only", lambda: dx.copy_(hx, non_blocking=True)), ("d2h only", lambda: hy.copy_(dy, non_blocking=True)), ("sequential", seq), ("concurrent", par)):
    for _ in range(3): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): f()
    torch.cuda.synchronize(); print(name, round((time.perf_counter() - t0) / 20 * 1e3, 3), "ms", flush=True)
