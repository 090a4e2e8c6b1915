import sys, os, time, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2210_03523_b200 as dg, workloads as W
mesh = W.cube_mesh(16); orders = W.orders_uniform(mesh.E, 6)
S = dg.Solver(mesh); S.set_orders(orders)
q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, center=W.cfg2_center(), sigma=0.08)).cuda()
qb, g, ref = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
tau = torch.empty((mesh.E, 3, 9), dtype=torch.float64, device="cuda")
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
ev = lambda: torch.cuda.Event(enable_timing=True)
for mode in ["steps", "loop"]:
    for it in range(4):
        if mode == "steps":
            S.rk_steps(50, q, qb, g, dts[0], dts[1], 0.5)
        else:
            a, b = q, qb
            for k in range(50):
                S.rk_step_dt(a, b, g, dts[k % 2], 0.5, dts[(k + 1) % 2]); a, b = b, a
        S.rhs_eval(q, ref); S.tau_estimate(q, ref, reference=dg.REF_SOLVER, tau=tau)
        e2 = ev(); e2.record()
        t0 = time.perf_counter()
        sel = S.select_orders(tau, 1e-4, 3, 8)[0]
        t1 = time.perf_counter()
        qn = S.transfer(sel, q)
        t2 = time.perf_counter()
        e3 = ev(); e3.record(); torch.cuda.synchronize()
        print(mode, it, "gpu e2->e3 ms", round(e2.elapsed_time(e3), 3), "cpu select ms", round((t1 - t0) * 1e3, 3), "cpu transfer ms", round((t2 - t1) * 1e3, 3))
