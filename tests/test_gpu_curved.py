"""GPU vs oracle parity on curved (extruded O-grid) meshes, Euler and
Navier-Stokes with BR1 (cfg4 / cfg5 structure, BASELINE.json B:10-11)."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import RES_TOL, TAU_TOL, rel_linf, tau_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2210_03523_b200 as m

    m.build()
    return m


def ogrid_case(name):
    nsp = W.ns_params()
    if name == "cfg4_small":  # cfg4 structure at reduced size: 8 x 16 x 1, g=4, N=4
        mesh = W.ogrid_mesh(8, 16, 1, ratio=1.1 ** 6, g_eta=4)
        orders = W.orders_uniform(mesh.E, 4)
    elif name == "cfg4_adapted":  # after static adaptation: mixed orders in [4,8] (mortars)
        mesh = W.ogrid_mesh(6, 12, 2, ratio=1.1 ** 8, g_eta=4)
        orders = W.orders_random(mesh.E, 4, 7, 41)
    elif name == "cfg4_full":  # BASELINE cfg4 [B:10] at full size: 48 x 64 x 1, g=4, N=4
        mesh = W.make_mesh(W.CONFIGS["cfg4"]["mesh"])
        orders = W.orders_uniform(mesh.E, 4)
    elif name == "cfg5_subbox":  # cfg5 structure: g=2, Nx,Ny ~ U{2..8}, Nz = 2
        mesh = W.ogrid_mesh(6, 16, 4, ratio=1.1 ** 4, g_eta=2)
        orders = W.orders_random(mesh.E, (2, 2, 2), (8, 8, 2), 5)
    else:
        raise KeyError(name)
    return mesh, orders, nsp


def setup(dg, orc, name, physics="ns"):
    import torch

    mesh, orders, nsp = ogrid_case(name)
    ph_o = orc.phys(orc.NS if physics == "ns" else orc.EULER, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    P = orc.Problem(mesh, ph_o)
    q = W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=4)
    S = dg.Solver(mesh, physics=dg.NS if physics == "ns" else dg.EULER, mu=nsp["mu"], Pr=nsp["Pr"],
                  qinf=nsp["qinf"])
    S.set_orders(orders)
    return mesh, orders, P, S, q, torch.from_numpy(q).cuda()


def test_node_coords_match(dg, orc):
    mesh, orders, P, S, q, qd = setup(dg, orc, "cfg4_small")
    assert np.abs(S.node_coords() - P.node_coords(orders)).max() < 1e-13 * 20


@pytest.mark.parametrize("name", ["cfg4_small", "cfg4_adapted", "cfg5_subbox", "cfg4_full"])
@pytest.mark.parametrize("physics", ["ns", "euler"])
@pytest.mark.parametrize("variant", [0, 1])
def test_curved_rhs_parity(dg, orc, name, physics, variant):
    mesh, orders, P, S, q, qd = setup(dg, orc, name, physics)
    r = S.rhs_eval(qd, variant=variant).cpu().numpy()
    ro = P.rhs(orders, q, variant)
    assert rel_linf(r, ro, orders) < RES_TOL


def test_curved_freestream_gpu(dg, orc):
    import torch

    mesh, orders, nsp = ogrid_case("cfg5_subbox")
    mesh.nbr[mesh.nbr == W.BC_WALL] = W.BC_FARFIELD
    orders = W.orders_random(mesh.E, (1, 3, 1), (8, 8, 3), 7)  # resolves the face metrics
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S.set_orders(orders)
    q = torch.from_numpy(W.uniform_state(orders, vel=(1.0, 0.0, 0.0), p=nsp["p_inf"])).cuda()
    r = S.rhs_eval(q).cpu().numpy()
    assert np.abs(r).max() < 1e-9  # |q| ~ 45 (energy)


def test_curved_conservation_periodic_ns(dg, orc):
    """Periodic curved-free case: NS on a periodic cube mapped through the
    curved path (gorder 2 geometry of an affine box forces the curved kernels)."""
    import torch

    m = W.cube_mesh(3)
    # lift the geometry to order 2 (same box): the mesh is no longer 'affine' for dg_mesh_upload
    g2 = np.empty((m.E, 3, 27))
    x2 = np.array([0.0, 0.5, 1.0])
    for e in range(m.E):
        lo = m.geo[e, :, 0]
        hi = np.array([m.geo[e, 0, 1], m.geo[e, 1, 2], m.geo[e, 2, 4]])
        for k in range(3):
            for j in range(3):
                for i in range(3):
                    idx = i + 3 * (j + 3 * k)
                    g2[e, :, idx] = lo + (hi - lo) * np.array([x2[i], x2[j], x2[k]])
    m.geo = g2
    m.gorder = (2, 2, 2)
    orders = W.orders_random(m.E, 2, 6, 13)
    ph = orc.phys(orc.NS, mu=0.01, Pr=0.72)
    P = orc.Problem(m, ph)
    X = P.node_coords(orders)
    q = W.pulse_state(X, orders, sigma=0.15)
    S = dg.Solver(m, physics=dg.NS, mu=0.01, Pr=0.72)
    S.set_orders(orders)
    qd = torch.from_numpy(q).cuda()
    r = S.rhs_eval(qd)
    ro = P.rhs(orders, q)
    assert rel_linf(r.cpu().numpy(), ro, orders) < RES_TOL
    sums, _ = S.diagnostics(qd, r)
    M = P.mass(orders)
    from test_gpu_parity import per_var
    ab = np.array([np.abs(a * M).sum() for a in per_var(r.cpu().numpy(), orders)])
    assert np.all(np.abs(sums) < 1e-13 * ab)


@pytest.mark.parametrize("name", ["cfg4_small", "cfg5_subbox", "cfg4_full"])
def test_curved_rk_dt(dg, orc, name):
    import torch

    mesh, orders, P, S, q, qd = setup(dg, orc, name)
    qa, qb, g = qd.clone(), torch.empty_like(qd), torch.empty_like(qd)
    dts = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2)]
    S.compute_dt(qa, 0.5, dts[0])
    qo = q.copy()
    for step in range(3):
        dto = P.dt(orders, qo, 0.5)
        assert abs(dts[step % 2].item() - dto) <= 1e-13 * dto
        S.rk_step_dt(qa, qb, g, dts[step % 2], 0.5, dts[(step + 1) % 2])
        qa, qb = qb, qa
        qo = P.rk3_step(orders, qo, dto)
    assert rel_linf(qa.cpu().numpy(), qo, orders) < RES_TOL


@pytest.mark.parametrize("name", ["cfg4_small", "cfg5_subbox", "cfg4_full"])
@pytest.mark.parametrize("ref", ["solver", "same"])
@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("kernel", ["grp", "ext", "generic"])
def test_curved_tau_parity(dg, orc, name, ref, form, kernel, monkeypatch):
    """Isolated tau on the extruded O-grids: k_tau_grp (an element's levels
    batched per CTA, the default on extruded meshes), k_tau_ext (one CTA per
    level, DGTAU_TAU_PERLEVEL=1; both with compact coarse metrics) and the
    generic 3-D k_tau_curved (DGTAU_TAU_GENERIC=1)."""
    if kernel == "generic":
        monkeypatch.setenv("DGTAU_TAU_GENERIC", "1")
    if kernel == "ext":
        monkeypatch.setenv("DGTAU_TAU_PERLEVEL", "1")
    mesh, orders, P, S, q, qd = setup(dg, orc, name)
    if ref == "solver":
        tg = S.tau_estimate(qd, S.rhs_eval(qd), formulation=form, reference=dg.REF_SOLVER).cpu().numpy()
        to = P.tau_estimate(orders, q, P.rhs(orders, q), form)
    else:
        tg = S.tau_estimate(qd, None, formulation=form, reference=dg.REF_SAME).cpu().numpy()
        to = P.tau_estimate(orders, q, P.rhs(orders, q, orc.ISOLATED), form)
    assert tau_rel(tg, to) < TAU_TOL


@pytest.mark.parametrize("name", ["cfg4_small", "cfg5_subbox"])
@pytest.mark.parametrize("form", [0, 1])
def test_curved_tau_noniso_parity(dg, orc, name, form):
    """Non-isolated tau (reading R7) on the curved NS meshes: coarse
    levels with walls, far field, BR1 and (cfg5) mortars."""
    mesh, orders, P, S, q, qd = setup(dg, orc, name)
    tg = S.tau_estimate(qd, S.rhs_eval(qd), formulation=form, reference=dg.REF_SOLVER, noniso=True).cpu().numpy()
    to = P.tau_estimate_noniso(orders, q, P.rhs(orders, q), form)
    assert tau_rel(tg, to) < TAU_TOL


@pytest.mark.parametrize("name", ["cfg4_small", "cfg5_subbox"])
@pytest.mark.parametrize("kernel", ["grp", "ext", "generic"])
def test_curved_tau_euler_parity(dg, orc, name, kernel, monkeypatch):
    """Euler on the curved extruded meshes: the tau kernels' inviscid branch."""
    if kernel == "generic":
        monkeypatch.setenv("DGTAU_TAU_GENERIC", "1")
    if kernel == "ext":
        monkeypatch.setenv("DGTAU_TAU_PERLEVEL", "1")
    mesh, orders, P, S, q, qd = setup(dg, orc, name, physics="euler")
    tg = S.tau_estimate(qd, S.rhs_eval(qd), reference=dg.REF_SOLVER).cpu().numpy()
    to = P.tau_estimate(orders, q, P.rhs(orders, q))
    assert tau_rel(tg, to) < TAU_TOL


@pytest.mark.parametrize("name", ["cfg4_small", "cfg5_subbox"])
def test_curved_tau_l2_restriction_parity(dg, orc, name):
    mesh, orders, P, S, q, qd = setup(dg, orc, name)
    tg = S.tau_estimate(qd, S.rhs_eval(qd), restriction=1).cpu().numpy()
    to = P.tau_estimate(orders, q, P.rhs(orders, q), restriction=1)
    assert tau_rel(tg, to) < TAU_TOL


def test_cfg4_static_adaptation_cycle(dg, orc):
    """Static p-adaptation (Fig. 2) on the cfg4 structure at reduced
    size: 3 estimation stages accumulated with approach 2 / F_max, one
    selection (rule b, N in [4,8]); orders exact; then the adapted layout
    (with mortars) advances in parity."""
    import torch

    mesh, orders, P, S, q, qd = setup(dg, orc, "cfg4_small")
    Nmin, Nmax, tmax = 4, 8, 1.0
    K = Nmax - Nmin + 1
    total_g = torch.zeros((mesh.E, K, K, K), dtype=torch.float64, device="cuda")
    total_o = np.zeros((mesh.E, K, K, K))
    qa, qb, g = qd.clone(), torch.empty_like(qd), torch.empty_like(qd)
    qo = q.copy()
    for stage in range(3):
        for _ in range(2):
            dto = P.dt(orders, qo, 0.5)
            dtg = torch.tensor([dto], dtype=torch.float64, device="cuda")
            S.rk_step(qa, qb, g, dtg)
            qa, qb = qb, qa
            qo = P.rk3_step(orders, qo, dto)
        to = P.tau_estimate(orders, qo, P.rhs(orders, qo))
        mp, _ = orc.build_map(orders, to, Nmin, Nmax)
        total_o = orc.combine_max(total_o, mp)
        S.select_orders(torch.from_numpy(to).cuda(), tmax, Nmin, Nmax, mode=dg.SELECT_STATIC_ACCUM, total_map=total_g)
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
    assert rel_linf(qd.cpu().numpy(), qo, orders) < RES_TOL
    r = S.rhs_eval(qd).cpu().numpy()
    assert rel_linf(r, P.rhs(orders, qo), orders) < RES_TOL


def test_full_size_cfg5_sampled(dg, orc):
    """BASELINE cfg5 [B:11] at FULL size (96 x 256 x 16 O-grid, 393,216
    elements, ~42.5 M DOF, orders Nx, Ny ~ U{2..8}, Nz = 2, NS): the device
    residual and tau-estimate of 48 sampled elements against the oracle on a
    local mesh around them -- the sampled elements and their face neighbours
    owned, the next ring as halo, which is everything the BR1 residual of a
    sampled element reads (the same construction that makes the multi-rank
    owned results exact, test_dist_gloo)."""
    import torch

    from paper_2210_03523_b200 import partition as part

    spec = W.CONFIGS["cfg5"]
    mesh = W.make_mesh(spec["mesh"])
    orders = W.make_orders(spec["orders"], mesh.E)
    nsp = W.ns_params()
    q = W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), noise=1e-3, seed=4)
    S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    S.set_orders(orders)
    qd = torch.from_numpy(q).cuda()
    rd = S.rhs_eval(qd)
    tg = S.tau_estimate(qd, rd).cpu().numpy()
    r = rd.cpu().numpy()
    del qd, rd
    rng = np.random.default_rng(55)
    samp = np.sort(rng.choice(mesh.E, 48, replace=False))
    nb = mesh.nbr[samp].ravel()
    ring = np.unique(nb[nb >= 0])
    owner = np.ones(mesh.E, np.int32)
    owner[samp] = 0
    owner[ring] = 0
    lm = part.local_mesh(mesh, owner, 0)
    lo = np.ascontiguousarray(orders[lm.gids], np.int32)
    off = W.offsets(orders, 5)
    ql = np.concatenate([q[off[g]:off[g + 1]] for g in lm.gids])
    ph_o = orc.phys(orc.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    Pl = orc.Problem(lm, ph_o)
    rl = Pl.rhs(lo, ql)
    tl = Pl.tau_estimate(lo, ql, rl)
    offl = W.offsets(lo, 5)
    pos = {int(g): i for i, g in enumerate(lm.gids)}
    li = np.array([pos[int(e)] for e in samp])
    r_g = np.concatenate([r[off[e]:off[e + 1]] for e in samp])
    r_o = np.concatenate([rl[offl[i]:offl[i + 1]] for i in li])
    assert rel_linf(r_g, r_o, orders[samp]) < RES_TOL
    assert tau_rel(tg[samp], tl[li]) < TAU_TOL


@pytest.mark.parametrize("name", ["cfg5_subbox", "cfg4_adapted"])
@pytest.mark.parametrize("physics", ["ns", "euler"])
def test_tau_grp_vs_perlevel(dg, orc, name, physics, monkeypatch):
    """k_tau_grp does the same operations per node and level as k_tau_ext
    (only the CTA batching differs); the compiler's fma contraction may differ
    between the two kernels, so they agree to a few ulp of the level maxima."""
    mesh, orders, P, S, q, qd = setup(dg, orc, name, physics=physics)
    r = S.rhs_eval(qd)
    tg = S.tau_estimate(qd, r).cpu().numpy()
    monkeypatch.setenv("DGTAU_TAU_PERLEVEL", "1")
    tl = S.tau_estimate(qd, r).cpu().numpy()
    assert np.array_equal(np.isnan(tg), np.isnan(tl))
    ok = ~np.isnan(tg)
    assert np.all(np.abs(tg[ok] - tl[ok]) <= 1e-13 * np.abs(tl[ok]).max())
