"""Wall-clock breakdown of the e2e (host b/x) solve at cfg2 vs the device-resident solve."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1604_07163_b200 import tmgx as T  # noqa: E402

np3 = (257, 257, 257)
torch.cuda.set_device(0)
w = T.World(1)
s = T.SolverNode(w, T.Problem(np3, 0), T.MGConfig(7, 2, T.EST_LANCZOS))
n = s.local_size()
cfg = T.KrylovConfig("cg", rtol=1e-8, initial_guess_nonzero=False)
bh = torch.empty(n, dtype=torch.float64, pin_memory=True)
xh = torch.zeros(n, dtype=torch.float64, pin_memory=True)
bh.numpy()[:] = s.rhs(1234)
bd = bh.cuda()
xd = torch.zeros_like(bd)


def wall(f, k=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, sum(ts) / k * 1e3


print("seeded device solve  min/mean ms: %.2f %.2f" % wall(lambda: s.solve_seeded(1234, cfg=cfg)))
print("device b/x solve     min/mean ms: %.2f %.2f" % wall(lambda: s.solve_ptr(bd.data_ptr(), xd.data_ptr(), True, cfg)))
print("host b/x solve       min/mean ms: %.2f %.2f" % wall(lambda: s.solve_ptr(bh.data_ptr(), xh.data_ptr(), False, cfg)))
rep = s.solve_ptr(bh.data_ptr(), xh.data_ptr(), False, cfg)
print("host solve device-timed ms: %.2f its %d" % (rep.t_solve_s * 1e3, rep.iterations))
