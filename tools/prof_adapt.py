"""Cost of one dynamic adaptation on the affine Euler path (host planning in
dg_set_orders, the first residual of a new layout, steady residuals, tau,
selection, transfer), cube meshes n^3 with random mixed orders.
usage: python tools/prof_adapt.py [--runtime] [n ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402


def ev_ms(fn, reps=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rt = "--runtime" in sys.argv
for n in [int(x) for x in sys.argv[1:] if not x.startswith("--")] or [8, 16, 24]:
    mesh = W.cube_mesh(n)
    S = dg.Solver(mesh, path=dg.PATH_RUNTIME if rt else dg.PATH_AUTO)
    res = {"n": n, "E": mesh.E, "path": "runtime" if rt else "auto"}
    o1 = W.orders_random(mesh.E, 2, 8, 1)
    o2 = W.orders_random(mesh.E, 2, 8, 2)
    S.set_orders(o1)
    q = torch.from_numpy(W.uniform_state(o1)).cuda()
    r = torch.empty_like(q)
    S.rhs_eval(q, r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.set_orders(o2)
    torch.cuda.synchronize()
    res["set_orders_ms"] = (time.perf_counter() - t0) * 1e3
    q2 = torch.from_numpy(W.uniform_state(o2)).cuda()
    r2 = torch.empty_like(q2)
    t0 = time.perf_counter()
    S.rhs_eval(q2, r2)
    torch.cuda.synchronize()
    res["first_rhs_ms_wall"] = (time.perf_counter() - t0) * 1e3
    res["rhs_ms"] = ev_ms(lambda: S.rhs_eval(q2, r2), 20)
    qb, g = torch.empty_like(q2), torch.empty_like(q2)
    dt = torch.full((1,), 1e-5, dtype=torch.float64, device="cuda")
    res["rk_step_ms"] = ev_ms(lambda: S.rk_step(q2, qb, g, dt), 20)
    res["tau_ms"] = ev_ms(lambda: S.tau_estimate(q2, r2), 5)
    tau = S.tau_estimate(q2, r2)
    t0 = time.perf_counter()
    sel, _ = S.select_orders(tau, 1e-4, 2, 8)
    res["select_ms_wall"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    qt = S.transfer(o1, q2)
    torch.cuda.synchronize()
    res["transfer_ms_wall"] = (time.perf_counter() - t0) * 1e3
    res["ndof"] = S.ndof
    res["buckets"] = int(len({tuple(x) for x in o2}))
    print(json.dumps(res), flush=True)
