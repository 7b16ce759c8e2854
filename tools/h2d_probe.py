"""Host<->device copy bandwidth on this box (pinned, 136 MB = one 257^3 fp64 vector)."""
import time

import torch

n = 257 ** 3
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.uniform_()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, f in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt*1e3:.2f} ms  {n*8/dt/1e9:.1f} GB/s")
# both directions concurrently on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"bidir: {dt*1e3:.2f} ms for 2 x {n*8/1e6:.0f} MB")
