"""ncu driver: NS O-grid configs (cfg4 / cfg5 / cfg5u): one RK step + one SOLVER tau-estimate."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
spec = W.CONFIGS["cfg5" if cfg == "cfg5u" else cfg]
mesh = W.make_mesh(spec["mesh"])
orders = W.orders_uniform(mesh.E, (8, 8, 2)) if cfg == "cfg5u" else W.make_orders(spec["orders"], mesh.E)
nsp = W.ns_params()
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=4)).cuda()
qb, g, r = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
S.rk_step_dt(q, qb, g, dts[0], 0.5, dts[1])
S.rhs_eval(qb, r)
S.tau_estimate(qb, r)
torch.cuda.synchronize()
print("ok", S.ndof)
