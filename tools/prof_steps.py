"""ncu driver: cfg2 layout, a few dg_rk_steps calls (trace-fed face passes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

mesh = W.cube_mesh(16)
orders = W.orders_uniform(mesh.E, 6)
S = dg.Solver(mesh)
S.set_orders(orders)
q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, center=W.cfg2_center(), sigma=0.08)).cuda()
qb, g = torch.empty_like(q), torch.empty_like(q)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
for _ in range(2):
    S.rk_steps(4, q, qb, g, dts[0], dts[1], 0.5)
torch.cuda.synchronize()
print("ok")
