"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the hot path once -- affine Euler uniform (cfg1) and mixed
orders (8^3, orders U{2..7}: mortars, graphs), curved NS (cfg5 recipe on a
6 x 16 x 4 sub-box: face kernels, element pipelines, tau) -- residuals, RK
steps, tau-estimates (isolated and non-isolated), selection, transfer."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(S, q):
    r = S.rhs_eval(q)
    S.rhs_eval(q, variant=1)
    dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S.compute_dt(q, 0.5, dts[0])
    qa, qb, g = q.clone(), torch.empty_like(q), torch.empty_like(q)
    S.rk_steps(2, qa, qb, g, dts[0], dts[1], 0.5)
    tau = S.tau_estimate(qa, S.rhs_eval(qa))
    S.tau_estimate(qa, None, reference=dg.REF_SAME)
    S.tau_estimate(qa, r, noniso=True)
    sel, _ = S.select_orders(tau, 1e-4, 1, 8)
    S.transfer(sel, qa)
    S.diagnostics(qa, r)
    torch.cuda.synchronize()


if which in ("all", "cube"):
    for orders_fn, n in ((lambda E: W.orders_uniform(E, 3), 4), (lambda E: W.orders_random(E, 2, 7, 3), 8)):
        mesh = W.cube_mesh(n)
        orders = orders_fn(mesh.E)
        S = dg.Solver(mesh)
        S.set_orders(orders)
        q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, sigma=0.15)).cuda()
        run(S, q)
        print("cube", n, "ok")
if which in ("all", "ns"):
    nsp = W.ns_params()
    mesh = W.ogrid_mesh(6, 16, 4, ratio=1.1 ** 4, g_eta=2)
    orders = W.make_orders(W.CONFIGS["cfg5"]["orders"], mesh.E)
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S.set_orders(orders)
    q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), seed=5)).cuda()
    run(S, q)
    print("ns ok")
