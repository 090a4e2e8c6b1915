"""Kernel-level timings (CUDA events, many reps) of the hot calls on a layout:
rhs non-isolated / isolated, RK stage (fused), tau-estimate."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--noniso", action="store_true", help="also time the non-isolated tau-estimation")
a = ap.parse_args()
if a.cfg in ("cfg4", "cfg5", "cfg5u"):
    pass
elif a.cfg == "cfg2":
    mesh = W.cube_mesh(16)
    orders = W.orders_uniform(mesh.E, 6)
    kw = dict(center=W.cfg2_center(), sigma=0.08)
elif a.cfg.startswith("uniform"):
    N = int(a.cfg[7:])
    mesh = W.cube_mesh(16)
    orders = W.orders_uniform(mesh.E, N)
    kw = dict(sigma=0.1)
else:
    mesh = W.cube_mesh(32)
    orders = W.orders_random(mesh.E, 2, 7, 3)
    kw = dict(sigma=0.1)
if a.cfg in ("cfg4", "cfg5", "cfg5u"):  # Navier-Stokes on the curved O-grid (B:10-11)
    spec = W.CONFIGS["cfg5" if a.cfg == "cfg5u" else a.cfg]
    mesh = W.make_mesh(spec["mesh"])
    orders = W.orders_uniform(mesh.E, (8, 8, 2)) if a.cfg == "cfg5u" else W.make_orders(spec["orders"], mesh.E)
    nsp = W.ns_params()
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S.set_orders(orders)
    q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=4)).cuda()
else:
    S = dg.Solver(mesh)
    S.set_orders(orders)
    q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, **kw)).cuda()
qb, g, r = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])


def timeit(fn, reps=a.reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


ndof = S.ndof
res = {"cfg": a.cfg, "ndof": ndof, "E": mesh.E}
res["rhs_noniso_us"] = timeit(lambda: S.rhs_eval(q, r, variant=0))
res["rhs_iso_us"] = timeit(lambda: S.rhs_eval(q, r, variant=1))
res["rk_step_us"] = timeit(lambda: S.rk_step_dt(q, qb, g, dts[0], 0.5, dts[1]))
res["tau_solver_us"] = timeit(lambda: S.tau_estimate(q, r), reps=max(3, a.reps // 4))
if a.noniso:
    S.tau_estimate(q, r, noniso=True)  # builds the coarse-level contexts once per layout
    res["tau_noniso_us"] = timeit(lambda: S.tau_estimate(q, r, noniso=True), reps=max(3, a.reps // 4))
res["rk_steps10_us"] = timeit(lambda: S.rk_steps(10, q, qb, g, dts[0], dts[1], 0.5), reps=max(3, a.reps // 4))
res["gdofs_rk_stage_traces"] = 30 * ndof / res["rk_steps10_us"] / 1e3
res["gdofs_rhs"] = ndof / res["rhs_noniso_us"] / 1e3
res["gdofs_rk_stage"] = 3 * ndof / res["rk_step_us"] / 1e3
res["tau_Melem_s"] = mesh.E / res["tau_solver_us"]
print(json.dumps(res))
