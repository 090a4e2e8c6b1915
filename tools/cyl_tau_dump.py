"""Dump the SOLVER tau (new and traditional) of the cfg4 cylinder run at a
few step counts (diagnosis of the map / sentinel behaviour, DESIGN R11).
usage: python tools/cyl_tau_dump.py --noise 0 --steps 80000 260000 --out gpurun_out/cyl_tau.npz"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--noise", type=float, default=0.0)
ap.add_argument("--steps", type=int, nargs="+", default=[80000])
ap.add_argument("--out", default="gpurun_out/cyl_tau.npz")
ap.add_argument("--ref", choices=("solver", "same"), default="solver")
a = ap.parse_args()
nsp = W.ns_params()
mesh = W.make_mesh(W.CONFIGS["cfg4"]["mesh"])
orders = W.orders_uniform(mesh.E, 4)
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=a.noise, seed=4)).cuda()
qb, g = torch.empty_like(q), torch.empty_like(q)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
out, done = {}, 0
for n in sorted(a.steps):
    S.rk_steps(n - done, q, qb, g, dts[0], dts[1], 0.5) if (n - done) % 2 == 0 else None
    done = n
    r = S.rhs_eval(q) if a.ref == "solver" else None
    refk = dg.REF_SOLVER if a.ref == "solver" else dg.REF_SAME
    out[f"s{n}_new"] = S.tau_estimate(q, r, formulation=dg.TAU_NEW, reference=refk).cpu().numpy()
    out[f"s{n}_trad"] = S.tau_estimate(q, r, formulation=dg.TAU_TRADITIONAL, reference=refk).cpu().numpy()
np.savez_compressed(a.out, **out)
print("ok", list(out))
