"""cfg5 (129^3 x 3 Q1 elasticity, 6 levels, V(2,2), rtol 1e-6) on one GPU with the layout
BASELINE configs[4] names for 8 GPUs: 8 boxes, telescope r = 8 at level 3 (all boxes on this
GPU, same-process region copies instead of NVLink), against the one-box solve. Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1604_07163_b200 import tmgx as T  # noqa: E402


def run(R, tele, reps=5):
    w = T.World(R)
    s = T.ElastSolver(w, (129,) * 3, 6, smooth_its=2, telescope=tele)
    b = s.rhs()
    cfg = T.KrylovConfig("cg", rtol=1e-6)
    for _ in range(2):
        x, rep = s.solve(b, cfg=cfg)
    ts = []
    for _ in range(reps):
        x, rep = s.solve(b, cfg=cfg)
        ts.append(rep.t_solve_s)
    return dict(R=R, telescope=[(t.level, t.reduction_factor) for t in tele], its=rep.iterations,
                ms=1e3 * min(ts), launches=rep.kernel_launches, xnorm=float(np.linalg.norm(x)))


if __name__ == "__main__":
    a = run(1, [])
    b = run(8, [T.TelescopeStage(3, 8)])
    print(json.dumps({"one_box": a, "cfg5_layout_8_boxes": b,
                      "xnorm_rel_diff": abs(a["xnorm"] - b["xnorm"]) / a["xnorm"]}))
