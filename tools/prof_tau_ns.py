"""ncu driver: one SOLVER tau-estimate on cfg5 (or cfg4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
spec = W.CONFIGS[cfg]
mesh = W.make_mesh(spec["mesh"])
orders = W.make_orders(spec["orders"], mesh.E)
nsp = W.ns_params()
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=5)).cuda()
r = S.rhs_eval(q)
S.tau_estimate(q, r)
torch.cuda.synchronize()
print("ok")
