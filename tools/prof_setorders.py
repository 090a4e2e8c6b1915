"""Host cost of a layout change: dg_set_orders and the first residual after it
(CUDA-graph capture of the new mixed layout), for the dynamic-adaptation loop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

for n in (8, 16):
    mesh = W.cube_mesh(n)
    S = dg.Solver(mesh)
    o0 = W.orders_random(mesh.E, 2, 8, 1)
    S.set_orders(o0)
    q = torch.from_numpy(W.uniform_state(o0)).cuda()
    S.rhs_eval(q)
    torch.cuda.synchronize()
    ts, tr, tr2 = [], [], []
    for k in range(5):
        o = W.orders_random(mesh.E, 2, 8, 10 + k)
        t0 = time.perf_counter()
        S.set_orders(o)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        qk = torch.from_numpy(W.uniform_state(o)).cuda()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        S.rhs_eval(qk)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        S.rhs_eval(qk)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        ts.append(t1 - t0); tr.append(t3 - t2); tr2.append(t4 - t3)
    print(f"{n}^3 E={mesh.E}: set_orders {np.median(ts)*1e3:.2f} ms, first rhs {np.median(tr)*1e3:.2f} ms, "
          f"second rhs {np.median(tr2)*1e3:.2f} ms")
