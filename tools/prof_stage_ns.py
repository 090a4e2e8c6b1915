"""ncu driver: warm-up RK step, then ONE RK3 step (3 stages) on cfg5 -- the
kernels of the last 3 stages are the ones to sum per stage (traffic).
--rksteps: the step through dg_rk_steps (state traces between stages)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

spec = W.CONFIGS["cfg5"]
mesh = W.make_mesh(spec["mesh"])
orders = W.make_orders(spec["orders"], mesh.E)
nsp = W.ns_params()
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=5)).cuda()
qb, g = torch.empty_like(q), torch.empty_like(q)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
if "--rksteps" in sys.argv:  # dg_rk_steps (stages 2-3 read the state traces the previous stage wrote)
    S.rk_steps(1, q, qb, g, dts[0], dts[1], 0.5)
    torch.cuda.synchronize()
    n0 = S.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.rk_steps(1, qb, q, g, dts[1], dts[0], 0.5)
    e1.record()
    torch.cuda.synchronize()
    print("launches of the measured step", S.launches - n0, "ms", e0.elapsed_time(e1))
else:
    S.rk_step_dt(q, qb, g, dts[0], 0.5, dts[1])
    torch.cuda.synchronize()
    n0 = S.launches
    S.rk_step_dt(qb, q, g, dts[1], 0.5, dts[0])
    torch.cuda.synchronize()
    print("launches of the measured step", S.launches - n0)
