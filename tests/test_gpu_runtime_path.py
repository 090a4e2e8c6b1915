"""The runtime-order kernel path on affine meshes (dg_set_path(DG_PATH_RUNTIME),
include/dgtau.h): the same discretisation as the order-specialised path,
through the class-batched element and face kernels of the curved path.
GPU (C-ABI) vs the CPU oracle with the tolerances of test_gpu_parity.py, and
Navier-Stokes on an affine mesh, which only this path runs."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import CASES, RES_TOL, TAU_TOL, rel_linf, tau_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2210_03523_b200 as m

    m.build()
    return m


def setup_rt(dg, orc, case, path=None):
    import torch

    mesh, orders, kw = CASES[case]()
    P = orc.Problem(mesh)
    q = W.pulse_state(P.node_coords(orders), orders, **kw)
    S = dg.Solver(mesh, path=dg.PATH_RUNTIME if path is None else path)
    S.set_orders(orders)
    return mesh, orders, P, S, q, torch.from_numpy(q).cuda()


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("variant", [0, 1])
def test_rhs_runtime_path(dg, orc, case, variant):
    mesh, orders, P, S, q, qd = setup_rt(dg, orc, case)
    n0 = S.launches
    r = S.rhs_eval(qd, variant=variant).cpu().numpy()
    assert rel_linf(r, P.rhs(orders, q, variant), orders) < RES_TOL
    # a handful of launches whatever the number of (N1,N2,N3) buckets
    assert S.launches - n0 <= 8


@pytest.mark.parametrize("case", ["cfg1", "cfg3_subbox_mixed", "ragged_1to8"])
def test_rk_steps_runtime_path(dg, orc, case):
    import torch

    mesh, orders, P, S, q, qd = setup_rt(dg, orc, case)
    dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S.compute_dt(qd, 0.5, dts[0])
    qo = q.copy()
    assert abs(dts[0].item() - P.dt(orders, qo, 0.5)) <= 1e-14 * dts[0].item()
    qa, qb, g = qd.clone(), torch.empty_like(qd), torch.empty_like(qd)
    qs, dt_next = S.rk_steps(3, qa, qb, g, dts[0], dts[1], 0.5)
    for _ in range(3):
        qo = P.rk3_step(orders, qo, P.dt(orders, qo, 0.5))
    assert rel_linf(qs.cpu().numpy(), qo, orders) < RES_TOL
    assert abs(dt_next.item() - P.dt(orders, qo, 0.5)) <= 1e-13 * dt_next.item()


@pytest.mark.parametrize("case", ["cfg3_subbox_mixed", "ragged_1to8", "all_order8"])
@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("noniso", [False, True])
def test_tau_runtime_path(dg, orc, case, form, noniso):
    mesh, orders, P, S, q, qd = setup_rt(dg, orc, case)
    tg = S.tau_estimate(qd, S.rhs_eval(qd), formulation=form, noniso=noniso).cpu().numpy()
    ro = P.rhs(orders, q)
    to = P.tau_estimate_noniso(orders, q, ro, form) if noniso else P.tau_estimate(orders, q, ro, form)
    assert tau_rel(tg, to) < TAU_TOL


def test_dynamic_loop_runtime_path(dg, orc):
    """Two adaptation cycles of Fig. 1 on the runtime path:
    estimate -> select -> transfer -> re-layout -> residual, orders exact."""
    mesh, orders, P, S, q, qd = setup_rt(dg, orc, "cfg3_subbox_mixed")
    for cycle in range(2):
        tg = S.tau_estimate(qd, S.rhs_eval(qd))
        sel_g, _ = S.select_orders(tg, 1e-3, 2, 8, jump_rule=dg.JUMP_B, dec_cap=1)
        to = P.tau_estimate(orders, q, P.rhs(orders, q))
        sel_o, _ = orc.select_dynamic(orders, to, mesh.nbr, 1e-3, 2, 8, rule=orc.JUMP_B, cap=1)
        assert np.array_equal(sel_g, sel_o)
        qd = S.transfer(sel_g, qd).clone()
        q = orc.transfer(orders, q, sel_o)
        orders = sel_o
        S.set_orders(orders)
        assert rel_linf(qd.cpu().numpy(), q, orders) < RES_TOL
        assert rel_linf(S.rhs_eval(qd).cpu().numpy(), P.rhs(orders, q), orders) < RES_TOL


def test_ns_on_affine_mesh(dg, orc):
    """Navier-Stokes (BR1) on an affine periodic cube with mixed
    orders: residual and tau against the oracle (the order-specialised path
    is Euler-only)."""
    import torch

    nsp = W.ns_params()
    mesh = W.cube_mesh(4, 3, 3)
    orders = W.orders_random(mesh.E, 2, 6, 17)
    P = orc.Problem(mesh, orc.phys(orc.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"]))
    q = W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-2, seed=7)
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"], path=dg.PATH_RUNTIME)
    S.set_orders(orders)
    qd = torch.from_numpy(q).cuda()
    rg = S.rhs_eval(qd)
    ro = P.rhs(orders, q)
    c = (1.4 * nsp["p_inf"]) ** 0.5
    assert rel_linf(rg.cpu().numpy(), ro, orders, floor=(1.0, c, c, c, nsp["p_inf"] / 0.4)) < RES_TOL
    assert tau_rel(S.tau_estimate(qd, rg).cpu().numpy(), P.tau_estimate(orders, q, ro)) < TAU_TOL


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("variant", [0, 1])
def test_rhs_bucketed_path(dg, orc, case, variant):
    """The order-specialised kernels forced on every layout (DG_PATH_BUCKETED;
    AUTO hands many-bucket layouts to the runtime-order kernels)."""
    mesh, orders, P, S, q, qd = setup_rt(dg, orc, case, dg.PATH_BUCKETED)
    r = S.rhs_eval(qd, variant=variant).cpu().numpy()
    assert rel_linf(r, P.rhs(orders, q, variant), orders) < RES_TOL


@pytest.mark.parametrize("case", ["cfg3_subbox_mixed", "ragged_1to8"])
def test_rk_and_tau_bucketed_path(dg, orc, case):
    import torch

    mesh, orders, P, S, q, qd = setup_rt(dg, orc, case, dg.PATH_BUCKETED)
    dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S.compute_dt(qd, 0.5, dts[0])
    qa, qb, g = qd.clone(), torch.empty_like(qd), torch.empty_like(qd)
    qs, _ = S.rk_steps(3, qa, qb, g, dts[0], dts[1], 0.5)
    qo = q.copy()
    for _ in range(3):
        qo = P.rk3_step(orders, qo, P.dt(orders, qo, 0.5))
    assert rel_linf(qs.cpu().numpy(), qo, orders) < RES_TOL
    tg = S.tau_estimate(qd, S.rhs_eval(qd), noniso=True).cpu().numpy()
    assert tau_rel(tg, P.tau_estimate_noniso(orders, q, P.rhs(orders, q))) < TAU_TOL


def test_auto_path_switches_per_layout(dg, orc):
    """AUTO: a uniform layout launches one order-specialised kernel per
    residual; a many-bucket layout of the same solver a handful of
    runtime-order launches; both against the oracle."""
    import torch

    mesh = W.cube_mesh(6)
    P = orc.Problem(mesh)
    S = dg.Solver(mesh)
    for orders in (W.orders_uniform(mesh.E, 4), W.orders_random(mesh.E, 2, 7, 5), W.orders_uniform(mesh.E, 3)):
        S.set_orders(orders)
        q = W.pulse_state(P.node_coords(orders), orders, sigma=0.15)
        qd = torch.from_numpy(q).cuda()
        n0 = S.launches
        r = S.rhs_eval(qd).cpu().numpy()
        assert rel_linf(r, P.rhs(orders, q), orders) < RES_TOL
        assert S.launches - n0 <= 8
