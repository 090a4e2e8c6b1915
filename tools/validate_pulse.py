"""Physics validation run: error vs NDOF of uniform orders
against dynamic tau-based p-adaptation on the advected density pulse.

The pulse IC (constant u, p; reading A20) is an exact travelling solution of
the Euler equations (an entropy wave), so the error at time T is measured
against the translated IC.  Uniform runs: N = Nmin..Nmax.  Dynamic runs
(Fig. 1): every `--every` RK steps a SOLVER-reference
tau-estimate, dynamic selection (tau_max, [Nmin, Nmax], jump rule, decrease
cap 1), transfer of the state and a new layout.  Reported per run: the
time-averaged NDOF, the final L_inf and RMS density errors, the
steps and the device time.  Everything runs through libdgtau on one GPU.

Static runs (Fig. 2, approach 2 / F_max): an estimation run from
N0 over [0, T] accumulates the total truncation-error map every `--every`
steps, one selection per tau_max gives the static layout, and the pulse is
then run over [0, T] on that fixed layout (the paper compares the NDOF of
the static and dynamic layouts).

Stepping: the CFL step of each layout is formed once (one host read per
layout) and kept on the device, so the RK steps between two adaptations
launch back to back; the device time therefore measures the residual work
plus the adaptation cost (estimate, selection, transfer, re-layout), which
is what the paper's CPU-time comparison weighs.

usage: python tools/validate_pulse.py [--n 8] [--T 0.25] > profiles/r01_validate_pulse.json
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
ap.add_argument("--n", type=int, default=8, help="elements per direction")
ap.add_argument("--T", type=float, default=0.25, help="final time")
ap.add_argument("--cfl", type=float, default=0.5)
ap.add_argument("--every", type=int, default=10, help="RK steps between adaptations")
ap.add_argument("--nmin", type=int, default=2)
ap.add_argument("--nmax", type=int, default=8)
ap.add_argument("--n0", type=int, default=8, help="initial orders of the dynamic runs (the IC resolved at N_max)")
ap.add_argument("--sigma", type=float, default=0.08)
ap.add_argument("--path", choices=("auto", "runtime"), default="auto", help="residual kernel path (dg_set_path)")
ap.add_argument("--phases", action="store_true", help="per-phase host wall times (adds a sync per phase)")
ap.add_argument("--only", choices=("all", "dynamic"), default="all")
a = ap.parse_args()

VEL = (1.0, 0.5, 0.25)
C0 = (0.5, 0.5, 0.5)
mesh = W.cube_mesh(a.n)
PATH = dg.PATH_RUNTIME if a.path == "runtime" else dg.PATH_AUTO
PHASES = a.phases


def exact(S, orders, t):
    c = tuple((C0[i] + VEL[i] * t) % 1.0 for i in range(3))
    return W.pulse_state(S.node_coords(), orders, center=c, sigma=a.sigma, vel=VEL)


def rho_err(q, qe, orders):
    off = W.offsets(orders, 5)
    errs = []
    for e in range(len(orders)):
        n = (off[e + 1] - off[e]) // 5
        errs.append(q[off[e]:off[e] + n] - qe[off[e]:off[e] + n])
    d = np.concatenate(errs)
    return float(np.abs(d).max()), float(np.sqrt(np.mean(d * d)))


def run(orders, tau_max=None, rule=dg.JUMP_B):
    """uniform / static (tau_max None) or dynamic run over [0, T].  The step
    size is the CFL step of the current layout, formed once per
    layout (the pulse translates at constant speed, so the CFL rate is
    constant between adaptations) and held on the device: the RK steps of an
    estimation interval launch back to back without a host round trip."""
    S = dg.Solver(mesh, path=PATH)
    S.set_orders(orders)
    q = torch.from_numpy(exact(S, orders, 0.0)).cuda()
    qb, g = torch.empty_like(q), torch.empty_like(q)
    dtd = torch.zeros(1, dtype=torch.float64, device="cuda")
    t, steps, ndof_t, adapts = 0.0, 0, 0.0, 0
    ph = {"rk": 0.0, "estimate_select": 0.0, "transfer": 0.0, "set_orders": 0.0, "dt": 0.0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dt = S.compute_dt(q, a.cfl, sync=True)
    dtd.fill_(dt)
    h = time.perf_counter()

    def lap(key):  # host wall time of a phase (device work synchronised at its end)
        nonlocal h
        if PHASES:
            torch.cuda.synchronize()
            n = time.perf_counter()
            ph[key] += (n - h) * 1e3
            h = n

    while t < a.T - 1e-14:
        for _ in range(a.every):
            if t + dt > a.T - 1e-14:  # last step lands on T
                dtd.fill_(a.T - t)
                S.rk_step(q, qb, g, dtd)
                q, qb = qb, q
                ndof_t += W.ndof(orders) * (a.T - t)
                t = a.T
                steps += 1
                break
            S.rk_step(q, qb, g, dtd)
            q, qb = qb, q
            t += dt
            steps += 1
            ndof_t += W.ndof(orders) * dt
        lap("rk")
        if tau_max is not None and t < a.T - 1e-14:
            tau = S.tau_estimate(q, S.rhs_eval(q))
            new, _ = S.select_orders(tau, tau_max, a.nmin, a.nmax, jump_rule=rule, dec_cap=1)
            lap("estimate_select")
            if not np.array_equal(new, orders):
                q = S.transfer(new, q).clone()
                lap("transfer")
                orders = new
                S.set_orders(orders)
                qb, g = torch.empty_like(q), torch.empty_like(q)
                adapts += 1
                lap("set_orders")
                dt = S.compute_dt(q, a.cfl, sync=True)
                dtd.fill_(dt)
                lap("dt")
    ev1.record()
    torch.cuda.synchronize()
    linf, rms = rho_err(q.cpu().numpy(), exact(S, orders, a.T), orders)
    return {"ndof_avg": ndof_t / a.T, "ndof_final": W.ndof(orders), "err_linf": linf, "err_rms": rms,
            "steps": steps, "adaptations": adapts, "device_ms": ev0.elapsed_time(ev1),
            **({"phases_ms": ph} if PHASES else {})}


def static_maps():
    """estimation run from N0 over [0, T]: the static total map (approach 2,
    F_max) accumulated every `every` steps"""
    orders = W.orders_uniform(mesh.E, a.n0)
    S = dg.Solver(mesh, path=PATH)
    S.set_orders(orders)
    q = torch.from_numpy(exact(S, orders, 0.0)).cuda()
    qb, g = torch.empty_like(q), torch.empty_like(q)
    K = a.nmax - a.nmin + 1
    tot = torch.zeros((mesh.E, K, K, K), dtype=torch.float64, device="cuda")
    t, steps, stages = 0.0, 0, 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dt = S.compute_dt(q, a.cfl, sync=True)
    dtd = torch.full((1,), dt, dtype=torch.float64, device="cuda")
    while t < a.T - 1e-14:
        S.rk_step(q, qb, g, dtd)
        q, qb = qb, q
        t += dt
        steps += 1
        if steps % a.every == 0:
            tau = S.tau_estimate(q, S.rhs_eval(q))
            S.select_orders(tau, 1.0, a.nmin, a.nmax, mode=dg.SELECT_STATIC_ACCUM, total_map=tot)
            stages += 1
    ev1.record()
    torch.cuda.synchronize()
    return S, tot, stages, ev0.elapsed_time(ev1)


out = {"what": "advected density pulse (exact entropy wave), error vs time-averaged NDOF",
       "mesh": f"{a.n}^3 periodic affine hexes", "T": a.T, "cfl": a.cfl, "sigma": a.sigma,
       "adapt_every": a.every, "path": a.path, "Nmin": a.nmin, "Nmax": a.nmax, "runs": []}
t0 = time.time()
for N in range(a.nmin, a.nmax + 1) if a.only == "all" else ():
    r = run(W.orders_uniform(mesh.E, N))
    out["runs"].append({"kind": "uniform", "N": N, **r})
for rule, name in ((dg.JUMP_B, "b"), (dg.JUMP_A, "a")) if a.only == "all" else ((dg.JUMP_B, "b"),):
    for tm in (1e-1, 1e-2, 1e-3, 1e-4):
        r = run(W.orders_uniform(mesh.E, a.n0), tau_max=tm, rule=rule)
        out["runs"].append({"kind": "dynamic", "tau_max": tm, "rule": name, **r})
if a.only != "all":
    print(json.dumps(out, indent=1))
    sys.exit(0)
S0, tot, stages, est_ms = static_maps()
dummy = torch.zeros((mesh.E, 3, 9), dtype=torch.float64, device="cuda")
dummy[:, :, 0] = 1.0
for tm in (1e-1, 1e-2, 1e-3, 1e-4):
    sel, _ = S0.select_orders(dummy, tm, a.nmin, a.nmax, mode=dg.SELECT_STATIC_FINAL, total_map=tot.clone(),
                              jump_rule=dg.JUMP_B)
    r = run(sel)
    dyn = [x for x in out["runs"] if x["kind"] == "dynamic" and x["rule"] == "b" and x["tau_max"] == tm][0]
    out["runs"].append({"kind": "static", "tau_max": tm, "rule": "b", "estimation_stages": stages,
                        "estimation_ms": est_ms, "ndof_static_over_dynamic": r["ndof_avg"] / dyn["ndof_avg"], **r})
out["host_s"] = time.time() - t0
print(json.dumps(out, indent=1))
