"""Multi-rank ABI pieces on one GPU: two ranks' local meshes (owned + halo)
in one process, halo exchange emulated by device copies between their
state vectors (no kernels wait on each other).  Owned results equal the
single-rank GPU results exactly and the oracle within tolerance."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import RES_TOL, rel_linf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2210_03523_b200 as m

    m.build()
    return m


def _copy_halos(solvers, plans, states):
    """states[r] <- peer owned ranges, following the exchange plans."""
    for r, pl in enumerate(plans):
        for peer, rruns in pl.recv.items():
            sruns = plans[peer].send[r]
            src = __import__("torch").cat([states[peer][a:b] for a, b in sruns])
            o = 0
            for a, b in rruns:
                states[r][a:b].copy_(src[o:o + b - a])
                o += b - a


def _copy_traces(solvers, tplans, states, ncomp):
    """Face-trace halo exchange (partition.TracePlan, dg_trace_copy): every
    rank packs the traces its peers read, each peer unpacks them into the face
    nodes of its halo copies (the device copy stands in for the NCCL send)."""
    import torch

    for r, pl in enumerate(tplans):
        for peer in sorted(pl.send):
            buf = torch.empty(max(1, pl.send_len[peer]), dtype=torch.float64, device="cuda")
            solvers[r].trace_copy(torch.from_numpy(pl.send[peer]).cuda(), states[r], ncomp, buf, 0)
            rp = tplans[peer]
            assert rp.recv_len[r] == pl.send_len[peer]
            solvers[peer].trace_copy(torch.from_numpy(rp.recv[r]).cuda(), states[peer], ncomp, buf, 1)


@pytest.mark.parametrize("halo", ["states", "traces"])
@pytest.mark.parametrize("case", ["cube_mixed", "ogrid_ns", "cube_rebalanced"])
def test_two_rank_emulated(dg, orc, case, halo):
    """halo = "traces": only partition-boundary face traces are exchanged and
    every other node of the halo copies is NaN -- the owned results are still
    bit-identical, so nothing reads beyond the traces."""
    import torch

    from paper_2210_03523_b200 import partition as part

    if case in ("cube_mixed", "cube_rebalanced"):
        mesh = W.cube_mesh(4, 4, 6)
        g_orders = W.orders_random(mesh.E, 2, 6, 31)
        # bitwise comparison across solvers of different bucket counts: one
        # kernel family for all (AUTO would pick per layout)
        kw = dict(path=dg.PATH_BUCKETED)
        P = orc.Problem(mesh)
        if case == "cube_rebalanced":  # adapted orders skewed to low z, DOF-balanced slabs (dist.rebalance)
            g_orders[np.arange(mesh.E) // 16 < 2] = np.minimum(g_orders[np.arange(mesh.E) // 16 < 2] + 2, 8)
            owner = part.dof_owner(mesh.dims, g_orders, 2, axis=2)
        else:
            owner = part.slab_owner(mesh.dims, 2, axis=2)
        q_g = W.pulse_state(P.node_coords(g_orders), g_orders, sigma=0.2)
    else:
        mesh = W.ogrid_mesh(4, 8, 2, ratio=1.1 ** 12, g_eta=2)
        g_orders = W.orders_random(mesh.E, (2, 2, 2), (6, 6, 2), 32)
        nsp = W.ns_params()
        kw = dict(physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
        P = orc.Problem(mesh, orc.phys(orc.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"]))
        q_g = W.freestream_noise_state(g_orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]))
        owner = part.slab_owner(mesh.dims, 2, axis=1)  # azimuthal slabs
    # single-rank reference on the GPU
    S0 = dg.Solver(mesh, **kw)
    S0.set_orders(g_orders)
    q0 = torch.from_numpy(q_g).cuda()
    qa0, qb0, g0 = q0.clone(), torch.empty_like(q0), torch.empty_like(q0)
    dts0 = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S0.compute_dt(qa0, 0.5, dts0[0])
    dt_init = dts0[0].item()
    for s in range(2):
        S0.rk_step_dt(qa0, qb0, g0, dts0[s % 2], 0.5, dts0[(s + 1) % 2])
        qa0, qb0 = qb0, qa0
    # two local meshes
    lms = [part.local_mesh(mesh, owner, r) for r in range(2)]
    solvers, plans, gplans, qa, qb, gg = [], [], [], [], [], []
    blocks = [q_g[a:b] for a, b in zip(W.offsets(g_orders)[:-1], W.offsets(g_orders)[1:])]
    for lm in lms:
        S = dg.Solver(lm, **kw)
        S.set_owned(lm.n_own)
        lo = g_orders[lm.gids]
        S.set_orders(lo)
        solvers.append(S)
        if halo == "states":
            plans.append(part.HaloPlan(lm, lo, 5))
            gplans.append(part.HaloPlan(lm, lo, 15))
        else:
            plans.append(part.TracePlan(lm, lo, 5))
            gplans.append(part.TracePlan(lm, lo, 15))
        x = torch.from_numpy(np.concatenate([blocks[g] if i < lm.n_own else np.full_like(blocks[g], np.nan)
                                             for i, g in enumerate(lm.gids)])).cuda()
        qa.append(x)
        qb.append(torch.empty_like(x))
        gg.append(torch.empty_like(x))
    # global dt = max over ranks of the rates
    lam = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(2)]
    for r in range(2):
        solvers[r].dt_accumulate(qa[r], lam[r])
    lmax = torch.maximum(lam[0], lam[1])
    dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    solvers[0].dt_finalize(lmax.clone(), 0.5, dts[0])
    assert dts[0].item() == dt_init  # MAX of per-rank rates == global max (bitwise)
    for s in range(2):
        src = [qa, qb, qa]
        dst = [qb, qa, qb]
        for r in range(2):
            lam[r].zero_()
        for k in range(3):
            if halo == "states":
                _copy_halos(solvers, plans, src[k])
            else:
                _copy_traces(solvers, plans, src[k], 5)
            flags = 0
            if case == "ogrid_ns":  # BR1: gradient pass, gradient halo refresh, then the flux pass
                for r in range(2):
                    solvers[r].gradient(src[k][r])
                if halo == "states":
                    _copy_halos(solvers, gplans, [S.gradient_buffer() for S in solvers])
                else:
                    _copy_traces(solvers, gplans, [S.gradient_buffer() for S in solvers], 15)
                flags = dg.FLAG_GRADIENT_READY
            for r in range(2):
                solvers[r].rk_stage(k, src[k][r], dst[k][r], gg[r], dts[s % 2], lam[r] if k == 2 else None, flags)
        lmax = torch.maximum(lam[0], lam[1])
        solvers[0].dt_finalize(lmax, 0.5, dts[(s + 1) % 2])
        qa, qb = qb, qa
    # owned parts equal the single-rank result bitwise (same kernels, same inputs)
    ref_blocks = qa0.cpu().numpy()
    off = W.offsets(g_orders)
    for r, lm in enumerate(lms):
        got = qa[r][: solvers[r].owned_len()].cpu().numpy()
        want = np.concatenate([ref_blocks[off[g]:off[g + 1]] for g in lm.gids[: lm.n_own]])
        assert np.array_equal(got, want), np.abs(got - want).max()
    # and the oracle within tolerance
    qo = q_g.copy()
    dto = P.dt(g_orders, qo, 0.5)
    for s in range(2):
        qo2 = P.rk3_step(g_orders, qo, dto)
        qo, dto = qo2, P.dt(g_orders, qo2, 0.5)
    assert rel_linf(qa0.cpu().numpy(), qo, g_orders) < RES_TOL
    # distributed selection pieces: select_local + jump sweeps with emulated exchange
    tau_g = torch.from_numpy(P.tau_estimate(g_orders, q_g, P.rhs(g_orders, q_g))).cuda()
    sel0, _ = S0.select_orders(tau_g, 1e-4, 2, 8)
    a, b = [], []
    for r, lm in enumerate(lms):
        t_loc = tau_g[torch.from_numpy(lm.gids).cuda()].contiguous()
        out = torch.empty((lm.E, 3), dtype=torch.int32, device="cuda")
        solvers[r].select_local(t_loc, 1e-4, 2, 8, out)
        a.append(out)
        b.append(torch.empty_like(out))
    oplans = [part.HaloPlan(lm, np.zeros((lm.E, 3), np.int32), 3) for lm in lms]
    changed = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(64):
        _copy_halos(solvers, oplans, [x.view(-1) for x in a])
        changed.zero_()
        for r in range(2):
            solvers[r].jump_sweep(a[r], b[r], 1, 8, changed)
        a, b = b, a
        if changed.item() == 0:
            break
    for r, lm in enumerate(lms):
        assert np.array_equal(a[r][: lm.n_own].cpu().numpy(), sel0[lm.gids[: lm.n_own]])


def test_distsolver_single_rank_matches_solver(dg, orc):
    """DistSolver composition (exchange calls, all-reduces, distributed
    selection) on a 1-rank gloo group: identical to the plain Solver."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2210_03523_b200 import partition as part
    from paper_2210_03523_b200.dist import DistSolver

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=0, world_size=1)
    mesh = W.cube_mesh(4, 4, 4)
    orders = W.orders_random(mesh.E, 2, 6, 41)
    P = orc.Problem(mesh)
    q = torch.from_numpy(W.pulse_state(P.node_coords(orders), orders, sigma=0.2)).cuda()
    S = dg.Solver(mesh)
    S.set_orders(orders)
    D = DistSolver(mesh, part.slab_owner(mesh.dims, 1), 0, 1)
    D.set_orders(orders)
    r1 = S.rhs_eval(q)
    r2 = D.rhs_eval(q.clone())
    assert torch.equal(r1, r2)
    dt1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    dt2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    S.compute_dt(q, 0.5, dt1)
    D.compute_dt(q, 0.5, dt2)
    assert torch.equal(dt1, dt2)
    tau = S.tau_estimate(q, r1)
    sel1, _ = S.select_orders(tau, 1e-4, 2, 8)
    sel2 = D.select_orders(tau, 1e-4, 2, 8)
    assert np.array_equal(sel1, sel2)


def test_rebalance_single_rank_nccl(dg, orc):
    """dist.rebalance end to end on a one-rank NCCL group (the all-to-all,
    the DistSolver rebuild and the halo refresh run; with one rank every
    element stays): the rebalanced solver's residual equals the plain
    solver's, bit for bit."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2210_03523_b200 import partition as part
    from paper_2210_03523_b200.dist import DistSolver, rebalance

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    created = not dist.is_initialized()
    if created:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    assert dist.get_world_size() == 1
    grp = dist.new_group(ranks=[0], backend="nccl")
    try:
        mesh = W.cube_mesh(3, 3, 4)
        o1 = W.orders_random(mesh.E, 2, 5, 3)
        o2 = W.orders_random(mesh.E, 2, 7, 4)
        P = orc.Problem(mesh)
        ds = DistSolver(mesh, part.slab_owner(mesh.dims, 1), 0, 1, group=grp)
        ds.set_orders(o1)
        q2 = torch.from_numpy(W.pulse_state(P.node_coords(o2), o2, sigma=0.2)).cuda()
        # the state is already at o2 (as after a transfer); o1's solver object is what rebalances
        nd, q_new = rebalance(ds, o2, q2)
        r_d = nd.rhs_eval(q_new)
        S = dg.Solver(mesh)
        S.set_orders(o2)
        r_s = S.rhs_eval(q2)
        assert torch.equal(q_new, q2)
        assert torch.equal(r_d, r_s)
        # the NCCL branch of DistSolver.select_orders (device all_gather of the owned orders), twice (cached layout)
        tau = S.tau_estimate(q2, r_s)
        sel_s, _ = S.select_orders(tau, 1e-4, 2, 8)
        for _ in range(2):
            assert np.array_equal(nd.select_orders(tau, 1e-4, 2, 8), sel_s)
    finally:
        dist.destroy_process_group(grp)
        if created:
            dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cube_mixed", "ogrid_ns"])
def test_two_rank_noniso_tau(dg, orc, case):
    """Non-isolated tau across ranks through
    dg_tau_level: per coarse level (d, p), phase 0 on both ranks, the level's
    BR1 gradient face traces exchanged (NS), phase 1.  Only face traces of the
    fine state cross the partition (the halo interiors hold a finite poison),
    and the owned tau equal the single-rank non-isolated tau bit for bit."""
    import torch

    from paper_2210_03523_b200 import partition as part

    if case == "cube_mixed":
        mesh = W.cube_mesh(4, 4, 6)
        g_orders = W.orders_random(mesh.E, 2, 6, 31)
        kw = dict(path=dg.PATH_BUCKETED)  # one kernel family on every solver (bitwise comparison)
        P = orc.Problem(mesh)
        q_g = W.pulse_state(P.node_coords(g_orders), g_orders, sigma=0.2)
        owner = part.slab_owner(mesh.dims, 2, axis=2)
    else:
        mesh = W.ogrid_mesh(4, 8, 2, ratio=1.1 ** 12, g_eta=2)
        g_orders = W.orders_random(mesh.E, (2, 2, 2), (6, 6, 2), 32)
        nsp = W.ns_params()
        kw = dict(physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
        q_g = W.freestream_noise_state(g_orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]))
        owner = part.slab_owner(mesh.dims, 2, axis=1)
    S0 = dg.Solver(mesh, **kw)
    S0.set_orders(g_orders)
    q0 = torch.from_numpy(q_g).cuda()
    r0 = S0.rhs_eval(q0)
    t0 = S0.tau_estimate(q0, r0, noniso=True).cpu().numpy()
    off = W.offsets(g_orders)
    qb = [q_g[a:b] for a, b in zip(off[:-1], off[1:])]
    rr = r0.cpu().numpy()
    rb = [rr[a:b] for a, b in zip(off[:-1], off[1:])]
    lms = [part.local_mesh(mesh, owner, r) for r in range(2)]
    solvers, qs, rs, taus = [], [], [], []
    for lm in lms:
        S = dg.Solver(lm, **kw)
        S.set_owned(lm.n_own)
        lo = g_orders[lm.gids]
        S.set_orders(lo)
        solvers.append(S)
        qs.append(torch.from_numpy(np.concatenate([qb[g] if i < lm.n_own else np.full_like(qb[g], 7.25)
                                                   for i, g in enumerate(lm.gids)])).cuda())
        rs.append(torch.from_numpy(np.concatenate([rb[g] if i < lm.n_own else np.full_like(rb[g], -3.5)
                                                   for i, g in enumerate(lm.gids)])).cuda())
    _copy_traces(solvers, [part.TracePlan(lm, g_orders[lm.gids], 5) for lm in lms], qs, 5)
    for r in range(2):
        taus.append(solvers[r].tau_estimate(qs[r], rs[r]))  # isolated prefill (slot 0, undefined entries)
    nmax = g_orders.max(axis=0)
    for d in range(3):
        for p in range(1, int(nmax[d])):
            levs = [solvers[r].tau_level(d, p, 0, qs[r], rs[r]) for r in range(2)]
            if case == "ogrid_ns":
                tplans = []
                for lm in lms:
                    oc = g_orders[lm.gids].copy()
                    oc[:, d] = np.minimum(oc[:, d], p)
                    tplans.append(part.TracePlan(lm, oc, 15))
                _copy_traces(levs, tplans, [lv.gradient_buffer() for lv in levs], 15)
            for r in range(2):
                solvers[r].tau_level(d, p, 1, tau=taus[r])
    for r, lm in enumerate(lms):
        got = taus[r][: lm.n_own].cpu().numpy()
        want = t0[lm.gids[: lm.n_own]]
        assert np.array_equal(got, want, equal_nan=True), np.nanmax(np.abs(got - want))


@pytest.mark.parametrize("case", ["cube_mixed_runtime", "ogrid_ns"])
def test_two_rank_split_faces(dg, orc, case):
    """The overlapped stage of DistSolver (DG_FLAG_FACES_INTERIOR, then the
    trace exchange, then DG_FLAG_FACES_HALO): before every
    interior-face call the halo copies of the state (and of the gradient) are
    reset to NaN, so the interior faces provably read no halo data; two RK
    steps give owned states bit-identical to the single-rank solver."""
    import torch

    from paper_2210_03523_b200 import partition as part

    if case == "cube_mixed_runtime":
        mesh = W.cube_mesh(4, 4, 6)
        g_orders = W.orders_random(mesh.E, 2, 6, 31)
        kw = dict(path=dg.PATH_RUNTIME)
        P = orc.Problem(mesh)
        q_g = W.pulse_state(P.node_coords(g_orders), g_orders, sigma=0.2)
        owner = part.slab_owner(mesh.dims, 2, axis=2)
    else:
        mesh = W.ogrid_mesh(4, 8, 2, ratio=1.1 ** 12, g_eta=2)
        g_orders = W.orders_random(mesh.E, (2, 2, 2), (6, 6, 2), 32)
        nsp = W.ns_params()
        kw = dict(physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
        q_g = W.freestream_noise_state(g_orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]))
        owner = part.slab_owner(mesh.dims, 2, axis=1)
    ns = case == "ogrid_ns"
    S0 = dg.Solver(mesh, **kw)
    S0.set_orders(g_orders)
    q0 = torch.from_numpy(q_g).cuda()
    qa0, qb0, g0 = q0.clone(), torch.empty_like(q0), torch.empty_like(q0)
    dt = torch.full((1,), 1e-4, dtype=torch.float64, device="cuda")
    for _ in range(2):
        S0.rk_step(qa0, qb0, g0, dt)
        qa0, qb0 = qb0, qa0
    lms = [part.local_mesh(mesh, owner, r) for r in range(2)]
    off = W.offsets(g_orders)
    blocks = [q_g[a:b] for a, b in zip(off[:-1], off[1:])]
    solvers, tq, tg, qa, qb, gg = [], [], [], [], [], []
    for lm in lms:
        S = dg.Solver(lm, **kw)
        S.set_owned(lm.n_own)
        lo = g_orders[lm.gids]
        S.set_orders(lo)
        solvers.append(S)
        tq.append(part.TracePlan(lm, lo, 5))
        tg.append(part.TracePlan(lm, lo, 15))
        x = torch.from_numpy(np.concatenate([blocks[g] if i < lm.n_own else np.full_like(blocks[g], np.nan)
                                             for i, g in enumerate(lm.gids)])).cuda()
        qa.append(x)
        qb.append(torch.empty_like(x))
        gg.append(torch.zeros_like(x))
    own = [S.owned_len() for S in solvers]
    for _ in range(2):
        src, dst = [qa, qb, qa], [qb, qa, qb]
        for k in range(3):
            for r in range(2):
                src[k][r][own[r]:] = float("nan")
            if ns:
                for r in range(2):
                    solvers[r].gradient(src[k][r], flags=dg.FLAG_FACES_INTERIOR)
                _copy_traces(solvers, tq, src[k], 5)
                for r in range(2):
                    solvers[r].gradient(src[k][r], flags=dg.FLAG_FACES_HALO)
                    solvers[r].gradient_buffer()[3 * own[r]:] = float("nan")
                    solvers[r].rk_stage(k, src[k][r], dst[k][r], gg[r], dt, None,
                                        dg.FLAG_GRADIENT_READY | dg.FLAG_FACES_INTERIOR)
                _copy_traces(solvers, tg, [S.gradient_buffer() for S in solvers], 15)
                for r in range(2):
                    solvers[r].rk_stage(k, src[k][r], dst[k][r], gg[r], dt, None,
                                        dg.FLAG_GRADIENT_READY | dg.FLAG_FACES_HALO)
            else:
                for r in range(2):
                    solvers[r].rk_stage(k, src[k][r], dst[k][r], gg[r], dt, None, dg.FLAG_FACES_INTERIOR)
                _copy_traces(solvers, tq, src[k], 5)
                for r in range(2):
                    solvers[r].rk_stage(k, src[k][r], dst[k][r], gg[r], dt, None, dg.FLAG_FACES_HALO)
        qa, qb = qb, qa
    ref = qa0.cpu().numpy()
    for r, lm in enumerate(lms):
        got = qa[r][: own[r]].cpu().numpy()
        want = np.concatenate([ref[off[g]:off[g + 1]] for g in lm.gids[: lm.n_own]])
        assert np.array_equal(got, want), np.nanmax(np.abs(got - want))


@pytest.mark.parametrize("physics", ["euler", "ns"])
def test_distsolver_overlap_single_rank(dg, orc, physics):
    """DistSolver(overlap=True) on a one-rank gloo group: the overlapped stage
    (interior faces, exchange, halo faces + element kernels) through its
    Python driver gives the plain solver's RK step bit for bit."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2210_03523_b200 import partition as part
    from paper_2210_03523_b200.dist import DistSolver

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=0, world_size=1)
    if physics == "euler":
        mesh = W.cube_mesh(4, 4, 4)
        orders = W.orders_random(mesh.E, 2, 6, 41)
        kw = dict(path=dg.PATH_RUNTIME)
        q = W.pulse_state(orc.Problem(mesh).node_coords(orders), orders, sigma=0.2)
    else:
        mesh = W.ogrid_mesh(4, 8, 2, ratio=1.1 ** 12, g_eta=2)
        orders = W.orders_random(mesh.E, (2, 2, 2), (6, 6, 2), 32)
        nsp = W.ns_params()
        kw = dict(physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
        q = W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]))
    S = dg.Solver(mesh, **kw)
    S.set_orders(orders)
    D = DistSolver(mesh, part.slab_owner(mesh.dims, 1), 0, 1, overlap=True, **kw)
    D.set_orders(orders)
    qd = torch.from_numpy(q).cuda()
    outs = []
    for step in (lambda a, b, g, dt, dn: S.rk_step_dt(a, b, g, dt, 0.5, dn),
                 lambda a, b, g, dt, dn: D.rk_step_dt(a, b, g, dt, 0.5, dn)):
        dt = torch.zeros(1, dtype=torch.float64, device="cuda")
        S.compute_dt(qd, 0.5, dt)
        dn = torch.zeros_like(dt)
        qa, qb, g = qd.clone(), torch.empty_like(qd), torch.empty_like(qd)
        step(qa, qb, g, dt, dn)
        outs.append((qb.cpu().numpy(), dn.item()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
