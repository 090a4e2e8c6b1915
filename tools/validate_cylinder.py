"""Cylinder validation run: the cfg4
NS case (O-grid 48 x 64 x 1, N = 4, Re 100, Ma 0.2, free stream + 1e-3
noise, reading A22) run to T_e through libdgtau; every T_e/10 a SOLVER
tau-estimate in BOTH formulations -- the new tau~ and the
traditional tau = M tau~ -- accumulated into two static total
maps (approach 2, F_max); at T_e one static selection per
threshold (rule b, N in [4, 8]) gives the adapted NDOF of each formulation
(the traditional-vs-new comparison of Fig. 9: the paper's
traditional tau_max 1e-1 / 1e-2 / 5e-3 and new tau~_max 1e2 / 1 / 1e-1 give
similar NDOF).  With tau~_max = 1 (the cfg4 reading) the run then
continues 100 steps on the adapted layout (reading A23: no restart).

Both tau references are accumulated in the same run (--ref both): the
solver's non-isolated residual (A4 default) and the isolated fine residual
(SAME), see DESIGN.md "Finding (cfg4 cylinder, SOLVER reference)".  --spinup
T runs T time units first at a low order (cheap steps) so that the
estimation window samples developed shedding, as the paper's T_e = 12 = two
shedding cycles does; the state is then transferred to N = 4.

usage: python tools/validate_cylinder.py [--Te 12] [--spinup 100] > profiles/r02_validate_cylinder.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--Te", type=float, default=12.0)
ap.add_argument("--cfl", type=float, default=0.5)
ap.add_argument("--stages", type=int, default=10)
ap.add_argument("--ref", choices=("solver", "same", "both"), default="both",
                help="tau reference: the solver's non-isolated residual (A4 default) or the isolated fine residual")
ap.add_argument("--spinup", type=float, default=0.0,
                help="time units run first at order --spinup-order (developed shedding before the estimation window)")
ap.add_argument("--spinup-order", type=int, default=2)
ap.add_argument("--noise", type=float, default=1e-3, help="IC noise amplitude (reading A22: 1e-3; 0 = smooth impulsive start)")
a = ap.parse_args()

nsp = W.ns_params()
mesh = W.make_mesh(W.CONFIGS["cfg4"]["mesh"])
orders = W.orders_uniform(mesh.E, 4)
S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
S.set_orders(orders)
spin = {}
if a.spinup > 0:  # spin-up at a low order (cheap steps), then the state is transferred to N = 4
    os_ = W.orders_uniform(mesh.E, a.spinup_order)
    S2 = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S2.set_orders(os_)
    q2 = torch.from_numpy(W.freestream_noise_state(os_, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=a.noise, seed=4)).cuda()
    qb2, g2 = torch.empty_like(q2), torch.empty_like(q2)
    d2 = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S2.compute_dt(q2, a.cfl, d2[0])
    t2, n2 = 0.0, 0
    h2 = time.time()
    while t2 < a.spinup:
        S2.rk_steps(200, q2, qb2, g2, d2[0], d2[1], a.cfl)
        t2 += 200 * d2[0].item()
        n2 += 200
    sums2, mn2 = S2.diagnostics(q2, S2.rhs_eval(q2))
    spin = {"T": t2, "order": a.spinup_order, "steps": n2, "host_s": time.time() - h2, "min_rho": mn2[0], "min_p": mn2[1]}
    q = S2.transfer(orders, q2).clone()
    del S2, q2, qb2, g2
else:
    q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=a.noise, seed=4)).cuda()
qb, g = torch.empty_like(q), torch.empty_like(q)
Nmin, Nmax = 4, 8
K = Nmax - Nmin + 1
REFS = ("solver", "same") if a.ref == "both" else (a.ref,)
tot = {(f, rf): torch.zeros((mesh.E, K, K, K), dtype=torch.float64, device="cuda")
       for f in (dg.TAU_NEW, dg.TAU_TRADITIONAL) for rf in REFS}
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, a.cfl, dts[0])
t, steps, stage = 0.0, 0, 0
chunk = 200
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
next_est = a.Te / a.stages
log = []
h0 = time.time()
while stage < a.stages:
    # advance in device-looped chunks of RK steps, then re-check the time
    S.rk_steps(chunk, q, qb, g, dts[0], dts[1], a.cfl)  # even: ends in q, next dt in dts[0]
    dt_last = dts[0].item()
    steps += chunk
    t += chunk * dt_last  # step sizes vary slowly: time from the last dt (reported)
    if t >= next_est:
        r = S.rhs_eval(q)
        for (f, rf) in tot:
            if rf == "same":
                tau = S.tau_estimate(q, None, formulation=f, reference=dg.REF_SAME)
            else:
                tau = S.tau_estimate(q, r, formulation=f)
            S.select_orders(tau, 1.0, Nmin, Nmax, mode=dg.SELECT_STATIC_ACCUM, total_map=tot[(f, rf)])
        sums, mn = S.diagnostics(q, r)
        log.append({"stage": stage + 1, "t": t, "steps": steps, "dt": dt_last, "min_rho": mn[0], "min_p": mn[1]})
        stage += 1
        next_est += a.Te / a.stages
ev1.record()
torch.cuda.synchronize()
dummy = torch.zeros((mesh.E, 3, 9), dtype=torch.float64, device="cuda")
dummy[:, :, 0] = 1.0
sel = {}
res = {"what": "cfg4 cylinder (Re 100, Ma 0.2): static tau-estimation, traditional vs new (Fig. 9)",
       "Te": a.Te, "stages": a.stages, "steps": steps, "device_ms": ev0.elapsed_time(ev1), "uniform_N4_ndof": S.ndof,
       "noise": a.noise, "reference": a.ref, "spinup": spin, "log": log, "thresholds": []}
nr = W.CONFIGS["cfg4"]["mesh"][1]
ring = np.arange(mesh.E) % nr  # element (i, j, k): radial index fastest
bands = [(0, nr // 3), (nr // 3, 2 * nr // 3), (2 * nr // 3, nr)]
for (f, name, ths), rf in ((x, rf) for x in ((dg.TAU_NEW, "new", (1e2, 1e1, 1.0, 1e-1)),
                                            (dg.TAU_TRADITIONAL, "traditional", (1e-1, 1e-2, 5e-3, 1e-3)))
                           for rf in REFS):
    for tm in ths:
        o, _ = S.select_orders(dummy, tm, Nmin, Nmax, mode=dg.SELECT_STATIC_FINAL, total_map=tot[(f, rf)].clone(),
                               jump_rule=dg.JUMP_B)
        res["thresholds"].append({"formulation": name, "reference": rf, "tau_max": tm, "ndof": W.ndof(o),
                                  "orders_hist": np.bincount(o.ravel(), minlength=9)[4:].tolist(),
                                  # Fig. 9's question: where the orders go (mean order, radial thirds: cylinder..far field)
                                  "mean_order_by_radial_band": [float(o[(ring >= lo) & (ring < hi), :2].mean())
                                                                for lo, hi in bands]})
        if name == "new" and tm == 1.0 and rf == REFS[-1]:
            sel = o
# continue on the adapted layout (tau~_max = 1)
q2 = S.transfer(sel, q).clone()
S.set_orders(sel)
qb2, g2 = torch.empty_like(q2), torch.empty_like(q2)
dts2 = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q2, a.cfl, dts2[0])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
S.rk_steps(100, q2, qb2, g2, dts2[0], dts2[1], a.cfl)
e1.record()
torch.cuda.synchronize()
sums, mn = S.diagnostics(q2, S.rhs_eval(q2))
res["adapted"] = {"tau_max": 1.0, "formulation": "new", "ndof": S.ndof, "steps": 100,
                  "device_ms": e0.elapsed_time(e1), "min_rho": mn[0], "min_p": mn[1]}
res["host_s"] = time.time() - h0
print(json.dumps(res, indent=1))
