"""One cfg5 elasticity solve bracketed by cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1604_07163_b200 import tmgx as T  # noqa: E402

torch.cuda.set_device(0)
w = T.World(1)
s = T.ElastSolver(w, (129, 129, 129), 6, smooth_its=2)
b = torch.from_numpy(s.rhs()).cuda()
x = torch.zeros_like(b)
cfg = T.KrylovConfig("cg", rtol=1e-6, initial_guess_nonzero=False)
s.solve_ptr(b.data_ptr(), x.data_ptr(), cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
rep = s.solve_ptr(b.data_ptr(), x.data_ptr(), cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("its", rep.iterations, "ms", rep.t_solve_s * 1e3)
