"""Small driver for ncu captures: cfg2 layout (or mixed cfg3) residual/RK/tau launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
if a.cfg == "cfg2":
    mesh = W.cube_mesh(16)
    orders = W.orders_uniform(mesh.E, 6)
    kw = dict(center=W.cfg2_center(), sigma=0.08)
else:
    mesh = W.cube_mesh(32)
    orders = W.orders_random(mesh.E, 2, 7, 3)
    kw = dict(sigma=0.1)
S = dg.Solver(mesh)
S.set_orders(orders)
q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, **kw)).cuda()
qb, g, r = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for _ in range(a.reps):
    S.compute_dt(q, 0.5)
    S.rk_step(q, qb, g, S._dt)
    q, qb = qb, q
    S.rhs_eval(q, r)
    S.tau_estimate(q, r)
torch.cuda.synchronize()
print("ok", S.ndof)
