"""Per-kernel device times of cfg5 RK steps (torch.profiler / CUPTI, not a
bench number) for A/B comparison of kernel variants; writes the state after
the steps to --save so variants can be compared to each other.
Usage: DGTAU_SO=... python tools/kernel_times.py [--steps 2] [--save f.pt] [--cfg cfg5]"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_03523_b200 as dg  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--save", default=None)
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--tau", action="store_true")
ap.add_argument("--euler", action="store_true", help="Euler (cfg2 / cfg3 are Euler configurations)")
a = ap.parse_args()
spec = W.CONFIGS[a.cfg]
mesh = W.make_mesh(spec["mesh"])
orders = W.make_orders(spec["orders"], mesh.E)
nsp = W.ns_params()
S = (dg.Solver(mesh) if a.euler else dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"]))
S.set_orders(orders)
q0 = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=5)).cuda()
q, qb, g = q0.clone(), torch.empty_like(q0), torch.empty_like(q0)
dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
S.compute_dt(q, 0.5, dts[0])
S.rk_steps(1, q, qb, g, dts[0], dts[1], 0.5)  # warm-up (graph capture etc.)
torch.cuda.synchronize()
q.copy_(q0)
S.compute_dt(q, 0.5, dts[0])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res, _ = S.rk_steps(a.steps, q, qb, g, dts[0], dts[1], 0.5)
e1.record()
torch.cuda.synchronize()
print(f"{a.cfg} {a.steps} RK3 steps (events, no profiler): {e0.elapsed_time(e1):.3f} ms")
if a.save:
    torch.save(res.cpu(), a.save)
q.copy_(q0)
S.compute_dt(q, 0.5, dts[0])
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    S.rk_steps(a.steps, q, qb, g, dts[0], dts[1], 0.5)
    if a.tau:
        S.tau_estimate(q, S.rhs_eval(q), reference=dg.REF_SOLVER)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name[:70]
        agg[k][0] += 1
        agg[k][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"{k:72s} n={n:4d} total_ms={t / 1e3:9.3f} avg_us={t / n:9.1f} share={100 * t / tot:5.1f}%")
print(f"TOTAL_ms {tot / 1e3:.3f}")
