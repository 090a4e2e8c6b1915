#!/usr/bin/env python
"""Benchmark of the B200 hot path on BASELINE.json configs[1] (cfg2):

  Euler density pulse, fp64, periodic cube 16^3 elements, fine N=(6,6,6),
  pulse centre seeded in [0.3,0.7]^3, width 0.08; dynamic p-adaptation with
  tau_estimate every 50 RK steps, tolerance 1e-4.

One bench STEP = one estimation interval of that run = every row of the hot
path once over the cfg2 layout:
  50 x (CFL dt on device + one Williamson RK3 step = 3 fused residual/RK-stage
  launches)  ->  reference residual (SOLVER, non-isolated)  ->  batched
  tau-estimation over all coarse orders  ->  dynamic order selection with the
  jump fixpoint  ->  projection of the state onto the selected orders.
The layout is kept at N=6 across steps so that every step does identical
work (the projected state is the step's adaptation output).

metric: DGSEM residual GDOF/s (fp64), whole job: NDOF x residual evaluations
in the step (151) / step time, all ranks.  Also reported: tau-estimation
elements/s and the residual-kernel roofline.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "DGSEM residual GDOF/s (fp64) + tau-estimation elems/s"
RK_PER_STEP = 50
CFL = 0.5
TAU_MAX = 1e-4
NMIN, NMAX = 3, 8


def load_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic_k_res_t.json")
    if os.path.exists(p):
        return json.load(open(p)).get("dram_bytes_per_launch")
    return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def load_fp64_peak():
    """Measured DFMA peak (tools/fp64_peak.cu on a B200, profiles/r01_fp64_peak.json), TFLOP/s."""
    p = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    best = None
    if os.path.exists(p):
        for line in open(p):
            d = json.loads(line)
            if d.get("kernel") == "dfma":
                best = max(best or 0.0, d["tflops"])
    return (best, "measured DFMA (profiles/r01_fp64_peak.json)") if best else (37.2, "nominal 148 SM x 64 FMA x 2 x 1.965 GHz")


def flops_model(N):
    """Algorithmic fp64 flops (FMA = 2) of the method steps of SURVEY 8(c).1 on
    affine hexes with isotropic order N (counted from the definitions, not
    from kernel code):
      residual per DOF: primitives + the three axis fluxes (33); D^N along each
      line of each axis for 5 variables, even-odd form L^2/2 multiply-adds per
      line plus 2 L adds (15 (L + 2) per node); strong-form lifting at the two
      line ends (3 flops per end); Roe flux per face point (130) times face
      points per DOF (3 L^2 / L^3); per-node combination and RK update (50).
      tau per element: for every level (d, p < N): per coarse node the
      interpolation of q and R along d (2 x 5 x 2 L), the three fluxes (33),
      the three axis derivatives (15 (L_d' + 2)) and the combination (30)."""
    L = N + 1
    per_dof = 33 + 15 * (L + 2) + 30.0 / L + 130.0 * 3 / L + 50
    tau = 0.0
    for p in range(1, N):
        nodes = (p + 1) * L * L
        tau += 3 * nodes * (20 * L + 33 + 5 * ((p + 1 + 2) + 2 * (L + 2)) + 30)
    return per_dof, tau


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cfg2_inputs(S):
    X = S.node_coords()
    return W.pulse_state(X, S.orders, center=W.cfg2_center(), sigma=0.08)


def make_solver(dg, mesh, orders):
    S = dg.Solver(mesh)
    S.set_orders(orders)
    return S


def run_gpu(args, rank, world):
    import torch

    import paper_2210_03523_b200 as dg

    dg.build()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    if world == 1:
        mesh = W.cube_mesh(16)
        orders = W.orders_uniform(mesh.E, 6)
        S = make_solver(dg, mesh, orders)
        ndof = S.ndof
        n_elem = mesh.E
        q0_host = cfg2_inputs(S)
        E_loc = mesh.E
        select = lambda tau: S.select_orders(tau, TAU_MAX, NMIN, NMAX, mode=dg.SELECT_DYNAMIC,  # noqa: E731
                                             jump_rule=dg.JUMP_B, dec_cap=1)[0]
        local = lambda sel: sel  # noqa: E731
        rk = S.rk_step_dt
        rhs = S.rhs_eval
        owned_len = S.state_len
        core = S
    else:
        # weak scaling: global periodic 16 x 16 x (16 N) cube, z-slabs of 16^3 elements per rank
        from paper_2210_03523_b200 import partition as part
        from paper_2210_03523_b200.dist import DistSolver

        mesh = W.cube_mesh(16, 16, 16 * world, L=(1.0, 1.0, float(world)))
        owner = part.slab_owner(mesh.dims, world, axis=2)
        D = DistSolver(mesh, owner, rank, world)
        orders_g = W.orders_uniform(mesh.E, 6)
        D.set_orders(orders_g)
        S = D.S
        ndof = int(np.prod(orders_g[D.lm.gids[: D.n_own]].astype(np.int64) + 1, axis=1).sum())
        n_elem = D.n_own
        X = S.node_coords()
        q0_host = W.pulse_state(X, D.local_orders, center=W.cfg2_center(), sigma=0.08, L=(1.0, 1.0, float(world)))
        E_loc = D.lm.E
        select = lambda tau: D.select_orders(tau, TAU_MAX, NMIN, NMAX, rule=dg.JUMP_B, dec_cap=1)  # noqa: E731
        local = lambda sel: sel[D.lm.gids]  # noqa: E731
        rk = D.rk_step_dt
        rhs = D.rhs_eval
        owned_len = D.owned_len()
        core = S
    q0 = torch.from_numpy(q0_host).to(dev)
    qa = q0.clone()
    qb = torch.empty_like(qa)
    g = torch.empty_like(qa)
    ref = torch.empty_like(qa)
    tau = torch.empty((E_loc, 3, 9), dtype=torch.float64, device=dev)
    qn_buf = torch.empty(5 * 9 ** 3 * E_loc, dtype=torch.float64, device=dev)  # adapted state, any orders <= 8
    dts = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(2)]
    if world == 1:
        S.compute_dt(qa, CFL, dts[0])  # first step's dt; later ones come fused from the RK kernel
    else:
        D.compute_dt(qa, CFL, dts[0])
    stream = torch.cuda.current_stream()
    cur = [0]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(timers=None):
        nonlocal qa, qb
        if world == 1:  # the 50 RK3 steps in one call (dg_rk_steps: stage-to-stage face traces)
            if timers:
                e0, e1 = ev(), ev()
                e0.record(stream)
            S.rk_steps(RK_PER_STEP, qa, qb, g, dts[cur[0]], dts[1 - cur[0]], CFL)
            if RK_PER_STEP % 2:
                cur[0] = 1 - cur[0]
                qa, qb = qb, qa
            if timers:
                e1.record(stream)
                timers["rk"].append((e0, e1))
        for _ in range(RK_PER_STEP if world > 1 else 0):
            if timers:
                e0, e1 = ev(), ev()
                e0.record(stream)
            rk(qa, qb, g, dts[cur[0]], CFL, dts[1 - cur[0]])
            cur[0] = 1 - cur[0]
            if timers:
                e1.record(stream)
                timers["rk"].append((e0, e1))
            qa, qb = qb, qa
        if timers:
            e0, e1 = ev(), ev()
            e0.record(stream)
        rhs(qa, ref)
        core.tau_estimate(qa, ref, reference=dg.REF_SOLVER, tau=tau)
        if timers:
            e1.record(stream)
            timers["tau"].append((e0, e1))
        if timers:
            e2 = ev()
            e2.record(stream)
        sel = select(tau)
        qn = core.transfer(local(sel), qa, out=qn_buf)
        if timers:
            e3 = ev()
            e3.record(stream)
            timers["adapt"].append((e2, e3))
        return sel, qn

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # timed region
    timers = {"rk": [], "tau": [], "adapt": []}
    launches0 = core.launches
    clocks = ClockSampler(dev.index)
    if rank == 0:
        clocks.start()
        time.sleep(0.5)  # let nvidia-smi start streaming before the timed region (NVML init stalls)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    start, end = ev(), ev()
    start.record(stream)
    for _ in range(args.steps):
        sel, qn = step(timers)
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    launches = core.launches - launches0
    total_ms = start.elapsed_time(end)
    rk_ms = sum(a.elapsed_time(b) for a, b in timers["rk"])
    tau_ms = sum(a.elapsed_time(b) for a, b in timers["tau"])
    adapt_ms = sum(a.elapsed_time(b) for a, b in timers["adapt"])
    if world > 1:
        t = torch.tensor([total_ms, rk_ms, tau_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, rk_ms, tau_ms = t.tolist()
    evals_per_step = 3 * RK_PER_STEP + 1
    value = world * ndof * evals_per_step * args.steps / (total_ms * 1e-3) / 1e9
    # roofline of the dominant kernel pair: one RK stage = k_face + k_res_t
    # algorithmic bytes per DOF: stage 1 reads q, writes g and q' (A_1 = 0: g
    # not read) = 120 B; stages 2-3 read q, g and write g, q' = 160 B.
    bytes_rk_step = ndof * (120 + 160 + 160)
    rk_count = RK_PER_STEP * args.steps
    achieved = bytes_rk_step * rk_count / (rk_ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    tau_elems = n_elem * args.steps / (tau_ms * 1e-3)

    # end-to-end through the public API with host buffers: H2D of the step's
    # input state from pinned memory, the step, D2H of the adapted state + orders
    e2e = None
    if not args.no_e2e:
        # Each step: H2D of the step's input state from pinned memory, the step,
        # D2H of its adapted state (+ the orders, already on the host).  The
        # copies run on a copy stream, double-buffered, overlapping the
        # neighbouring steps' compute; every byte still crosses PCIe each step.
        pinned = torch.from_numpy(q0_host[:owned_len]).pin_memory()
        out_pinned = [torch.empty(qn_buf.numel(), dtype=torch.float64).pin_memory() for _ in range(2)]
        bufs = [torch.empty_like(qa) for _ in range(2)]
        qn_bufs = [qn_buf, torch.empty_like(qn_buf)]
        cs = torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(args.steps + 1)]
        ev_step = [torch.cuda.Event() for _ in range(args.steps)]
        ev_out = [torch.cuda.Event() for _ in range(args.steps)]
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(stream)
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            bufs[0][:owned_len].copy_(pinned, non_blocking=True)
        ev_in[0].record(cs)
        d2h = 0
        for k in range(args.steps):
            if k + 1 < args.steps:  # input of step k+1 while step k runs
                if k >= 1:
                    cs.wait_event(ev_step[k - 1])
                with torch.cuda.stream(cs):
                    bufs[(k + 1) % 2][:owned_len].copy_(pinned, non_blocking=True)
                ev_in[k + 1].record(cs)
            stream.wait_event(ev_in[k])
            if k >= 2:
                stream.wait_event(ev_out[k - 2])  # qn_bufs[k % 2] drained to the host
            qa = bufs[k % 2]
            qn_buf = qn_bufs[k % 2]
            sel, qn = step()
            ev_step[k].record(stream)
            cs.wait_event(ev_step[k])
            with torch.cuda.stream(cs):
                out_pinned[k % 2][: qn.numel()].copy_(qn, non_blocking=True)
            ev_out[k].record(cs)
            d2h += qn.numel() * 8 + sel.nbytes
        stream.wait_stream(cs)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        e2e = {"value": world * ndof * evals_per_step * args.steps / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": int(owned_len * 8), "d2h_bytes_per_step": int(d2h // args.steps),
               "copies": "pinned H2D of each step's input and D2H of its adapted state on a copy stream, "
                         "double-buffered, overlapping the neighbouring steps"}

    return dict(value=value, total_ms=total_ms, rk_ms=rk_ms, tau_ms=tau_ms, adapt_ms=adapt_ms, ndof=ndof, E=n_elem,
                achieved=achieved, peak=peak, peak_kind=peak_kind, tau_elems=tau_elems, clocks=clk,
                launches=launches, e2e=e2e, rk_count=rk_count, bytes_rk_step=bytes_rk_step)


def oracle_baseline(sample_rk_steps=1, with_tau=True):
    """The CPU oracle as it stands on this host's cores: a bounded sample of
    the same workload (cfg2 layout): RK3 steps + one tau-estimate."""
    import oracle

    mesh = W.cube_mesh(16)
    orders = W.orders_uniform(mesh.E, 6)
    P = oracle.Problem(mesh)
    X = P.node_coords(orders)
    q = W.pulse_state(X, orders, center=W.cfg2_center(), sigma=0.08)
    ndof = W.ndof(orders)
    t0 = time.perf_counter()
    for _ in range(sample_rk_steps):
        dt = P.dt(orders, q, CFL)
        q = P.rk3_step(orders, q, dt)
    t1 = time.perf_counter()
    tau_s = None
    if with_tau:
        r = P.rhs(orders, q)
        P.tau_estimate(orders, q, r)
        tau_s = time.perf_counter() - t1
    gdofs = ndof * 3 * sample_rk_steps / (t1 - t0) / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    return dict(value=gdofs, seconds=t1 - t0, tau_s=tau_s, tau_elems=mesh.E / tau_s if tau_s else None, cores=cores,
                sample=f"{sample_rk_steps} RK3 step(s) (3 residuals each) on the cfg2 layout (16^3 elements, N=6, "
                       f"{ndof} DOF)" + (" + 1 SOLVER residual + 1 tau-estimate" if with_tau else ""))


def fp64_block(res):
    """Secondary rooflines: algorithmic fp64 rate (flops_model) of the RK stage
    and of the tau-estimation against the measured DFMA peak."""
    peak, src = load_fp64_peak()
    per_dof, tau_el = flops_model(6)
    stage_tf = per_dof * res["ndof"] * 3 * res["rk_count"] / (res["rk_ms"] * 1e-3) / 1e12
    tau_tf = tau_el * res["tau_elems"] / 1e12
    return {"peak_tflops": peak, "peak_source": src,
            "rk_stage": {"flops_per_dof": round(per_dof, 1), "achieved_tflops": stage_tf, "frac": stage_tf / peak},
            "tau": {"flops_per_element": round(tau_el), "achieved_tflops": tau_tf, "frac": tau_tf / peak,
                    "note": "tau time includes the SOLVER reference residual"},
            "model": "bench.py flops_model (SURVEY 8(c).1 steps, FMA = 2)"}


def config_block(world, extra=None):
    c = {"workload": ("cfg2" if world == 1 else f"cfg2 per rank (weak scaling, global 16x16x{16 * world})") +
                     ": Euler density pulse, periodic 16^3 affine hexes, N=(6,6,6) Gauss-Lobatto, "
                     "50 RK3 steps (CFL 0.5) + SOLVER-reference tau-estimate + dynamic select (tau_max 1e-4, "
                     "N in [3,8], jump rule b, decrease cap 1) + transfer per step",
         "elements": 4096, "orders": [6, 6, 6], "ndof": 4096 * 343, "residuals_per_step": 3 * RK_PER_STEP + 1,
         "l2": "inputs larger than L2: each RK stage touches q, g, q' = 3 x 56.2 MB = 169 MB > 126 MB L2",
         "parallelism": f"domain decomposition dp{world}: z-slabs of 16^3 elements per rank, NCCL halo "
                        f"exchange per RK stage, MAX all-reduce of the CFL rate per step" if world > 1 else "single"}
    if extra:
        c.update(extra)
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        if args.impl == "ours":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group(backend=backend)

    if args.impl == "reference":
        if rank != 0:
            return
        # The reference arm for this tier is the CPU oracle, timed as it stands.
        import oracle

        oracle.build()
        for _ in range(args.warmup):
            oracle_baseline(1, with_tau=False)
        ts = []
        for _ in range(args.steps):
            r = oracle_baseline(1, with_tau=False)
            ts.append(r["seconds"])
        total = sum(ts)
        ndof = 4096 * 343
        value = ndof * 3 * args.steps / total / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GDOF/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_block(1, {"reference_step": "1 RK3 step (3 residuals) per step, CPU oracle"}),
                "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": r["cores"], "kind": "oracle",
                                 "sample": r["sample"]},
                "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    res = run_gpu(args, rank, world)
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle

        oracle.build()
        cb = oracle_baseline(1, with_tau=True)
        cpu = {"value": cb["value"], "unit": "GDOF/s", "cores": cb["cores"], "kind": "oracle", "sample": cb["sample"],
               "tau_elems_per_s": cb["tau_elems"]}
    line = {
        "metric": METRIC,
        "value": res["value"], "unit": "GDOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["total_ms"] / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(world),
        "tau_elems_per_s": res["tau_elems"] * world,
        "phase_ms_per_step": {"rk3_x50": res["rk_ms"] / args.steps, "ref_rhs_plus_tau": res["tau_ms"] / args.steps,
                              "select_plus_transfer": res["adapt_ms"] / args.steps},
        "rhs_rk_gdof_s": world * res["ndof"] * 3 * res["rk_count"] / (res["rk_ms"] * 1e-3) / 1e9,
        "roofline": {"kernel": "RK stage = k_face (face Riemann fluxes) + k_res_t (volume, lifting, fused RK update)",
                     "bound": "hbm", "achieved": res["achieved"],
                     "peak": res["peak"], "unit": "GB/s", "frac": res["achieved"] / res["peak"],
                     "peak_source": res["peak_kind"], "traffic": load_traffic(),
                     "bytes_per_dof": "120 (stage 1) / 160 (stages 2,3)"},
        "roofline_fp64": fp64_block(res),
        "cpu_baseline": cpu,
        "e2e": res["e2e"],
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
