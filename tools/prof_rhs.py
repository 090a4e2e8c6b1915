"""ncu driver: a few cfg2 non-isolated rhs evaluations (k_res_t<6,6,6> mode 0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

mesh = W.cube_mesh(16)
orders = W.orders_uniform(mesh.E, int(sys.argv[1]) if len(sys.argv) > 1 else 6)
S = dg.Solver(mesh)
S.set_orders(orders)
q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, center=W.cfg2_center(), sigma=0.08)).cuda()
r = torch.empty_like(q)
for _ in range(3):
    S.rhs_eval(q, r)
torch.cuda.synchronize()
print("ok")
