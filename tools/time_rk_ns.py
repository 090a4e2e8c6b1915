"""CUDA-event time of dg_rk_steps on cfg5 (ms per RK3 step) and of one
non-isolated residual: the quick check of a kernel change before a bench.
usage: python tools/time_rk_ns.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
spec = W.CONFIGS["cfg5"]
mesh = W.make_mesh(spec["mesh"])
orders = W.make_orders(spec["orders"], mesh.E)
nsp = W.ns_params()
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=5)).cuda()
qb, g, r = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
S.rk_steps(2, q, qb, g, dts[0], dts[1], 0.5)
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
torch.cuda.synchronize()
e0.record()
S.rk_steps(n, q, qb, g, dts[0], dts[1], 0.5)
e1.record()
for _ in range(5):
    S.rhs_eval(q, r)
e2.record()
torch.cuda.synchronize()
print(json.dumps({"ndof": S.ndof, "ms_per_rk_step": e0.elapsed_time(e1) / n, "ms_per_rhs": e1.elapsed_time(e2) / 5,
                  "rhs_gdofs": S.ndof / (e1.elapsed_time(e2) / 5) / 1e6}))
