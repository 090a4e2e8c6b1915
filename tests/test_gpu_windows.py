"""Trajectory parity windows of SURVEY 8(c) ("Parity criteria"), GPU through
the C ABI against the CPU oracle at BASELINE.json's full sizes:

* cfg2: the dynamic loop of Fig. 1 -- 50 RK3 steps, SOLVER
  tau-estimate, selection from the GPU's OWN tau, transfer, re-layout
  (dg_set_orders), 50 more steps; orders exact, the decisive margins (A15)
  reported;
* cfg3: 20 RK3 steps in the bench's launch configuration + one estimate and
  selection;
* cfg4: the static cycle of Fig. 2 at full size with a reduced
  step count: three estimation stages (approach 2, F_max), one selection,
  the adapted layout then advances;
* cfg5: the 16 x 32 x 4 sub-box run of the cfg5 recipe (NS, mixed orders,
  mortars on every face class): RK steps + estimate + selection.
Tolerances: relative L_inf 1e-11 on states (free-stream scales as floors,
reading R5), 1e-9 on tau, exact integer orders [B:5].
"""
import math

import numpy as np
import pytest

import workloads as W
from test_gpu_parity import EULER_PULSE_SCALES, RES_TOL, TAU_TOL, rel_linf, tau_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2210_03523_b200 as m

    m.build()
    return m


def ns_scales(nsp):
    """free-stream scales (rho, rho c x 3, p / (gamma - 1)) of the NS configs"""
    c = math.sqrt(1.4 * nsp["p_inf"])
    return (1.0, c, c, c, nsp["p_inf"] / 0.4)


def _advance(S, P, orders, qa, qo, nsteps, floor):
    """nsteps RK3 steps: GPU in one dg_rk_steps call (dt formed on the
    device), oracle step by step with its own dt; returns the new pair."""
    import torch

    dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S.compute_dt(qa, 0.5, dts[0])
    qb, g = torch.empty_like(qa), torch.empty_like(qa)
    qs, _ = S.rk_steps(nsteps, qa, qb, g, dts[0], dts[1], 0.5)
    for _ in range(nsteps):
        qo = P.rk3_step(orders, qo, P.dt(orders, qo, 0.5))
    assert rel_linf(qs.cpu().numpy(), qo, orders, floor=floor) < RES_TOL
    return qs.clone(), qo


def test_window_cfg2_dynamic_loop(dg, orc):
    """BASELINE cfg2 [B:8] at full size (16^3, N=6, tau_max 1e-4, N in [3,8],
    rule b, cap 1): 50 steps -> GPU tau -> GPU selection from the GPU tau ->
    transfer -> dg_set_orders -> 50 steps.  Orders identical to the oracle's
    own loop; every element's decisive margin is reported."""
    import torch

    mesh = W.cube_mesh(16)
    orders = W.orders_uniform(mesh.E, 6)
    P = orc.Problem(mesh)
    q = W.pulse_state(P.node_coords(orders), orders, center=W.cfg2_center(), sigma=0.08)
    S = dg.Solver(mesh)
    S.set_orders(orders)
    qa, qo = _advance(S, P, orders, torch.from_numpy(q).cuda(), q.copy(), 50, EULER_PULSE_SCALES)
    rg = S.rhs_eval(qa)
    tg = S.tau_estimate(qa, rg)
    ro = P.rhs(orders, qo)
    to = P.tau_estimate(orders, qo, ro)
    assert tau_rel(tg.cpu().numpy(), to) < TAU_TOL
    sel_g, mg = S.select_orders(tg, 1e-4, 3, 8, mode=dg.SELECT_DYNAMIC, jump_rule=dg.JUMP_B, dec_cap=1)
    sel_o, mo = orc.select_dynamic(orders, to, mesh.nbr, 1e-4, 3, 8, rule=orc.JUMP_B, cap=1)
    print(f"cfg2 window: min decisive margin GPU {mg.min():.3e} oracle {mo.min():.3e}; "
          f"NDOF {W.ndof(orders)} -> {W.ndof(sel_o)}")
    assert np.array_equal(sel_g, sel_o)
    assert not np.array_equal(sel_o, orders)  # the adaptation changes the layout
    qd = S.transfer(sel_g, qa)
    qo = orc.transfer(orders, qo, sel_o)
    orders = sel_o
    S.set_orders(orders)
    assert rel_linf(qd.cpu().numpy(), qo, orders, floor=EULER_PULSE_SCALES) < RES_TOL
    _advance(S, P, orders, qd, qo, 50, EULER_PULSE_SCALES)


def test_window_cfg3(dg, orc):
    """BASELINE cfg3 [B:9] at full size (32^3, orders U{2..7}, ~97 % mortar
    faces): 20 RK3 steps (one estimation interval), SOLVER tau, selection."""
    import torch

    mesh = W.cube_mesh(32)
    orders = W.orders_random(mesh.E, 2, 7, 3)
    P = orc.Problem(mesh)
    q = W.pulse_state(P.node_coords(orders), orders, sigma=0.1)
    S = dg.Solver(mesh)
    S.set_orders(orders)
    qa, qo = _advance(S, P, orders, torch.from_numpy(q).cuda(), q.copy(), 20, EULER_PULSE_SCALES)
    tg = S.tau_estimate(qa, S.rhs_eval(qa))
    to = P.tau_estimate(orders, qo, P.rhs(orders, qo))
    assert tau_rel(tg.cpu().numpy(), to) < TAU_TOL
    sel_g, _ = S.select_orders(tg, 1e-4, 1, 8, mode=dg.SELECT_DYNAMIC, jump_rule=dg.JUMP_B, dec_cap=1)
    sel_o, _ = orc.select_dynamic(orders, to, mesh.nbr, 1e-4, 1, 8, rule=orc.JUMP_B, cap=1)
    assert np.array_equal(sel_g, sel_o)


def test_window_cfg4_static_full(dg, orc):
    """BASELINE cfg4 [B:10] at full size (48 x 64 x 1 O-grid, N=4, NS Re 100):
    the static cycle of Fig. 2 with a reduced step count (three estimation
    stages of 4 RK steps each, approach 2 / F_max, tau_max 1, N in [4,8], rule
    b), orders exact, then 3 RK steps of the adapted (mortar) layout."""
    import torch

    nsp = W.ns_params()
    mesh = W.make_mesh(W.CONFIGS["cfg4"]["mesh"])
    orders = W.orders_uniform(mesh.E, 4)
    P = orc.Problem(mesh, orc.phys(orc.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"]))
    q = W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=4)
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S.set_orders(orders)
    fl = ns_scales(nsp)
    Nmin, Nmax, tmax = 4, 8, 1.0
    K = Nmax - Nmin + 1
    total_g = torch.zeros((mesh.E, K, K, K), dtype=torch.float64, device="cuda")
    total_o = np.zeros((mesh.E, K, K, K))
    qa, qo = torch.from_numpy(q).cuda(), q.copy()
    for stage in range(3):
        qa, qo = _advance(S, P, orders, qa, qo, 4, fl)
        tg = S.tau_estimate(qa, S.rhs_eval(qa))
        to = P.tau_estimate(orders, qo, P.rhs(orders, qo))
        assert tau_rel(tg.cpu().numpy(), to) < TAU_TOL
        mp, _ = orc.build_map(orders, to, Nmin, Nmax)
        total_o = orc.combine_max(total_o, mp)
        S.select_orders(tg, tmax, Nmin, Nmax, mode=dg.SELECT_STATIC_ACCUM, total_map=total_g)
    sel_o, _ = orc.select_from_map(total_o, Nmin, Nmax, tmax)
    sel_o, _ = orc.jump_fixpoint(mesh.nbr, sel_o, orc.JUMP_B, Nmax)
    dummy = torch.zeros((mesh.E, 3, 9), dtype=torch.float64, device="cuda")
    dummy[:, :, 0] = 1.0
    sel_g, _ = S.select_orders(dummy, tmax, Nmin, Nmax, mode=dg.SELECT_STATIC_FINAL, total_map=total_g)
    assert np.array_equal(sel_g, sel_o)
    qd = S.transfer(sel_g, qa)
    qo = orc.transfer(orders, qo, sel_o)
    orders = sel_o
    S.set_orders(orders)
    assert rel_linf(qd.cpu().numpy(), qo, orders, floor=fl) < RES_TOL
    _advance(S, P, orders, qd, qo, 3, fl)


def test_window_cfg5_subbox(dg, orc):
    """The cfg5 recipe [B:11] on a 16 x 32 x 4 sub-box (A21: g_eta = 2,
    radial ratio sqrt(1.1), N_x, N_y ~ U{2..8}, N_z = 2, NS): 5 RK3 steps,
    SOLVER tau, the dynamic selection of the bench (tau_max 1, N in [1,8])."""
    import torch

    nsp = W.ns_params()
    mesh = W.ogrid_mesh(16, 32, 4, ratio=math.sqrt(1.1), g_eta=2)
    orders = W.make_orders(W.CONFIGS["cfg5"]["orders"], mesh.E)
    P = orc.Problem(mesh, orc.phys(orc.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"]))
    q = W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=5)
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S.set_orders(orders)
    qa, qo = _advance(S, P, orders, torch.from_numpy(q).cuda(), q.copy(), 5, ns_scales(nsp))
    tg = S.tau_estimate(qa, S.rhs_eval(qa))
    to = P.tau_estimate(orders, qo, P.rhs(orders, qo))
    assert tau_rel(tg.cpu().numpy(), to) < TAU_TOL
    sel_g, mg = S.select_orders(tg, 1.0, 1, 8, mode=dg.SELECT_DYNAMIC, jump_rule=dg.JUMP_B, dec_cap=1)
    sel_o, _ = orc.select_dynamic(orders, to, mesh.nbr, 1.0, 1, 8, rule=orc.JUMP_B, cap=1)
    print(f"cfg5 sub-box: min decisive margin {mg.min():.3e}")
    assert np.array_equal(sel_g, sel_o)
