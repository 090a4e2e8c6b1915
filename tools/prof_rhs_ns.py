"""ncu driver: one non-isolated NS residual (after a warm-up one) on cfg4 /
cfg5 / cfg5u; the profiled launches are the last residual's (use
--launch-skip with the count printed by a dry run, or filter by NVTX-free
kernel name)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = W.CONFIGS["cfg5" if cfg == "cfg5u" else cfg]
mesh = W.make_mesh(spec["mesh"])
orders = W.orders_uniform(mesh.E, (8, 8, 2)) if cfg == "cfg5u" else W.make_orders(spec["orders"], mesh.E)
nsp = W.ns_params()
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=5)).cuda()
r = torch.empty_like(q)
torch.cuda.synchronize()
n0 = S.launches
for _ in range(reps):
    S.rhs_eval(q, r)
torch.cuda.synchronize()
print("launches per rhs", (S.launches - n0) // reps, "ndof", S.ndof)
